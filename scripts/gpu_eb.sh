cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
C=1:1024,3:1024,5:1024,1:148,1:65536,3:65536,5:262144
timeout 900 python scripts/exp_lib_ab.py $D scripts/lib_eb8.so $C > gpurun_out/ab_eb.log 2>&1
timeout 900 python scripts/exp_lib_ab.py scripts/lib_eb19.so $D $C >> gpurun_out/ab_eb.log 2>&1
