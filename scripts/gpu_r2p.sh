cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or full_size or decrypt_valid or small_batch or striding" > gpurun_out/pytest_wd.log 2>&1; echo "exit $?" >> gpurun_out/pytest_wd.log
timeout 900 python scripts/sweep_launch.py split 4194304 1 > gpurun_out/sweep_split_wd.log 2>&1
