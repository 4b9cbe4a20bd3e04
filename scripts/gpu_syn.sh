cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
timeout 600 python scripts/exp_lib_ab.py scripts/lib_syn2.so $D 1:1024,3:1024,5:1024,1:148,3:16384,5:8192 > gpurun_out/ab_syn.log 2>&1
timeout 600 python scripts/exp_lib_ab.py scripts/lib_synF.so $D 1:1024,3:1024,5:1024,1:148,3:16384,5:8192 >> gpurun_out/ab_syn.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_batch or variants" > gpurun_out/pytest_syn.log 2>&1; echo "exit $?" >> gpurun_out/pytest_syn.log
