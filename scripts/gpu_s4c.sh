# session 4: RM argmax by tournament — parity (quick GPU suite) and A/B against HQC_RM_TOURNAMENT=0
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not scaling_config and not round_trip_at_scale" > gpurun_out/pytest_tour.log 2>&1; echo "exit $?" >> gpurun_out/pytest_tour.log
C=3:65536,1:65536,5:262144,1:1024,3:1024,5:1024,3:4194304
timeout 900 python scripts/exp_lib_ab.py scripts/libx_notour.so paper_2512_12904_b200/libhqcgpu.so $C > gpurun_out/ab_tour.log 2>&1
