set -x
python -m pytest tests/test_gpu_parity.py -q -x -k "variants and 10" 2>&1 | tail -3
L=paper_2512_12904_b200/libhqcgpu.so
python scripts/exp_lib_ab.py KERNEL=1@$L KERNEL=10@$L 5:262144,5:65536,5:32768,1:65536,3:65536 2>&1
HQC_DEC_SPLIT=0 python scripts/exp_lib_ab.py KERNEL=1@$L KERNEL=10@$L 5:524288 2>&1
