cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
timeout 600 python scripts/exp_lib_ab.py scripts/lib_u1.so scripts/lib_u2.so 5:262144,3:65536,1:65536 > gpurun_out/ab_unroll.log 2>&1
timeout 600 python scripts/exp_lib_ab.py scripts/lib_u3.so $D 5:262144,3:65536,1:65536 >> gpurun_out/ab_unroll.log 2>&1
timeout 600 python scripts/exp_s1_ab.py scripts/lib_u1.so scripts/lib_u2.so s1:5:65536,s1:3:65536,s1:1:65536 > gpurun_out/ab_unroll_s1.log 2>&1
timeout 600 python scripts/exp_s1_ab.py scripts/lib_u3.so $D s1:5:65536,s1:3:65536,s1:1:65536 >> gpurun_out/ab_unroll_s1.log 2>&1
