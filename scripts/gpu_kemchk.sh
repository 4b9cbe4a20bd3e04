cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kem.py tests/test_gpu_encrypt.py -q -x -k "not scaling_config" > gpurun_out/pytest_kem2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_kem2.log
timeout 300 python scripts/prof_kem.py --levels 1,3,5 > gpurun_out/kem_prof2.log 2>&1
