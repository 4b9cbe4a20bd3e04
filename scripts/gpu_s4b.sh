# session 4: REDUX syndromes A/B and phase counters after riBM
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
C=1:1024,3:1024,5:1024,1:148,1:1,3:16384,1:32768,5:16384
timeout 900 python scripts/exp_lib_ab.py paper_2512_12904_b200/libhqcgpu.so scripts/libx_synr.so $C > gpurun_out/ab_synr.log 2>&1
timeout 300 python scripts/exp_sb_phases.py run > gpurun_out/sb_phases_ribm.log 2>&1
