cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_batch or striding or adversarial_quarters or edges" > gpurun_out/pytest_bm.log 2>&1; echo "exit $?" >> gpurun_out/pytest_bm.log
timeout 600 python scripts/exp_sb_phases.py run > gpurun_out/sb_phases3.log 2>&1
timeout 900 python scripts/exp_lib_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_exp_bm0.so 1:1024,3:1024,5:1024,3:65536,3:262144 > gpurun_out/ab_bm.log 2>&1
