cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encrypt.py tests/test_gpu_kem.py -m gpu -q -x > gpurun_out/pytest_enc3.log 2>&1; echo "exit $?" >> gpurun_out/pytest_enc3.log
timeout 600 python scripts/time_encrypt.py > gpurun_out/time_enc3.log 2>&1
