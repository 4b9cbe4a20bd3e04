cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/sweep_launch.py small > gpurun_out/sweep_small.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kem.py -m gpu -q -x > gpurun_out/pytest_kem.log 2>&1; echo "exit $?" >> gpurun_out/pytest_kem.log
