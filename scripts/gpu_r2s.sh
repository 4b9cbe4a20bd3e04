cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/pytest_sp.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sp.log
timeout 900 python scripts/exp_lib_ab.py KERNEL=7@paper_2512_12904_b200/libhqcgpu.so KERNEL=5@paper_2512_12904_b200/libhqcgpu.so 1:1,1:148,1:512,1:1024,1:2048,1:4096,3:1024,3:4096,5:1024,5:4096 > gpurun_out/ab_sp.log 2>&1
