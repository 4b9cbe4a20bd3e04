cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_batch or striding or decrypt_valid or variants" > gpurun_out/pytest_sb.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sb.log
timeout 900 python scripts/sweep_launch.py small > gpurun_out/sweep_small.log 2>&1
timeout 900 python scripts/sweep_launch.py split > gpurun_out/sweep_split.log 2>&1
