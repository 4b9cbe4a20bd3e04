cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/exp_lib_ab.py scripts/libhqc_exp_w1m8.so paper_2512_12904_b200/libhqcgpu.so 5:65536,5:262144 > gpurun_out/ab_w1m.log 2>&1
timeout 900 python scripts/exp_lib_ab.py scripts/libhqc_exp_w1m10.so scripts/libhqc_exp_w1m8.so 5:262144 >> gpurun_out/ab_w1m.log 2>&1
