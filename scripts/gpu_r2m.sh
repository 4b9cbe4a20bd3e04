cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_batch or striding or decrypt_valid or adversarial_quarters or edges or variants or full_size_config" > gpurun_out/pytest_sbpipe.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sbpipe.log
timeout 900 python scripts/exp_lib_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_prev.so 1:1024,3:1024,5:1024,3:16384,3:65536,3:262144 > gpurun_out/ab_sbpipe.log 2>&1
