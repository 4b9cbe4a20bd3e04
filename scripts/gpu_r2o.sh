cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/pytest_wd.log 2>&1; echo "exit $?" >> gpurun_out/pytest_wd.log
timeout 900 python scripts/exp_lib_ab.py KERNEL=6@paper_2512_12904_b200/libhqcgpu.so KERNEL=1@paper_2512_12904_b200/libhqcgpu.so 1:65536,1:262144,5:65536,5:262144,3:65536 > gpurun_out/ab_wd.log 2>&1
