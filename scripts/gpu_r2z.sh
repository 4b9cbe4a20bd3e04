cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/exp_lib_ab.py scripts/libhqc_exp_wdg18.so scripts/libhqc_exp_wdg20.so 1:65536,1:262144 > gpurun_out/ab_wdg.log 2>&1
timeout 900 python scripts/exp_lib_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libhqc_exp_wdg20.so 1:65536,1:262144 >> gpurun_out/ab_wdg.log 2>&1
