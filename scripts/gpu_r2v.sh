cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage1 or product" > gpurun_out/pytest_s1d.log 2>&1; echo "exit $?" >> gpurun_out/pytest_s1d.log
timeout 900 python scripts/exp_s1_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_prev.so s1:1:65536,s1:3:65536,s1:1:1024 > gpurun_out/ab_s1d.log 2>&1
