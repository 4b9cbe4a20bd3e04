cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_encrypt.py -m gpu -q -x -k "stage1 or product or small_batch or decrypt_valid or adversarial_quarters or edges or encrypt_matches or keygen or edge_supports" > gpurun_out/pytest_k1pipe.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k1pipe.log
timeout 900 python scripts/exp_s1_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_prev.so s1:1:65536,s1:3:65536,s1:5:65536 > gpurun_out/ab_k1pipe.log 2>&1
