# session 4: the warp-RS radius test
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_warp_rs.py -q > gpurun_out/pytest_warp_rs.log 2>&1; echo "exit $?" >> gpurun_out/pytest_warp_rs.log
