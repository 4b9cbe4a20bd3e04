cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
HQC_S1_KERNEL=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stage1 or stage2" > gpurun_out/pytest_s1p.log 2>&1; echo "exit $?" >> gpurun_out/pytest_s1p.log
for r in 1 2; do for K in 1 2; do echo "K$K $(HQC_S1_KERNEL=$K timeout 150 python scripts/time_s1_lib.py paper_2512_12904_b200/libhqcgpu.so 1,3,5)" >> gpurun_out/exp.log; done; done
