cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage1 or product" > gpurun_out/pytest_s1.log 2>&1; echo "exit $?" >> gpurun_out/pytest_s1.log
for L in 1 3 5; do timeout 300 python scripts/prof_kernels.py --level $L --only s1n --iters 20; done > gpurun_out/time_s1n.log 2>&1
