cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
timeout 600 python scripts/exp_lib_ab.py scripts/lib_vl0.so $D 3:65536,3:262144,3:4194304 > gpurun_out/ab_vl2.log 2>&1
HQC_DEC_KERNEL=8 timeout 300 python scripts/time_kind.py 1:65536,5:262144 >> gpurun_out/ab_vl2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or valid or adversarial or full_size" > gpurun_out/pytest_vl2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_vl2.log
