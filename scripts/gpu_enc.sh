cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_encrypt.py tests/test_gpu_kem.py -q -x > gpurun_out/pytest_enc.log 2>&1; echo "exit $?" >> gpurun_out/pytest_enc.log
timeout 300 python scripts/prof_kem.py --levels 1,3,5 > gpurun_out/kem_prof.log 2>&1
HQC_ENC_KERNEL=1 timeout 300 python scripts/prof_kem.py --levels 3 > gpurun_out/kem_prof_old.log 2>&1
