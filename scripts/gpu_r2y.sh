cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stage1 or product or small_batch or decrypt_valid or adversarial_quarters or edges or striding or full_size_config" > gpurun_out/pytest_ref.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ref.log
timeout 900 python scripts/exp_s1_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_prev.so dec:1:65536,dec:3:65536,dec:5:262144,dec:1:1024,s1:1:65536,s1:3:65536,s1:5:65536 > gpurun_out/ab_refactor.log 2>&1
