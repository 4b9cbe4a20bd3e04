cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
C=1:1024,3:1024,5:1024,1:148,3:16384
timeout 600 python scripts/exp_lib_ab.py $D scripts/lib_wF.so $C > gpurun_out/ab_wrs.log 2>&1
timeout 600 python scripts/exp_lib_ab.py scripts/lib_wB.so scripts/lib_wFB.so $C >> gpurun_out/ab_wrs.log 2>&1
