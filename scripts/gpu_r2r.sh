cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage3 or rs or decrypt_valid or adversarial_quarters or edges or variants or small_batch" > gpurun_out/pytest_gexp.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gexp.log
timeout 900 python scripts/exp_lib_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_prev.so 1:65536,3:65536,5:262144,1:1024 > gpurun_out/ab_gexp.log 2>&1
