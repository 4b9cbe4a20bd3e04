# session 4: riBM in the warp RS decoder — parity (quick GPU suite) and A/B against HQC_BM_RIBM=0
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not scaling_config and not round_trip_at_scale" > gpurun_out/pytest_ribm.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ribm.log
C=1:1024,3:1024,5:1024,1:148,1:1,3:16384,1:32768,5:16384
timeout 900 python scripts/exp_lib_ab.py scripts/libx_noribm.so paper_2512_12904_b200/libhqcgpu.so $C > gpurun_out/ab_ribm.log 2>&1
