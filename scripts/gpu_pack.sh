cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
timeout 600 python scripts/exp_lib_ab.py $D scripts/lib_pack.so 3:65536,3:1024,3:262144 > gpurun_out/ab_pack.log 2>&1
timeout 600 python scripts/exp_s1_ab.py $D scripts/lib_pack.so s1:3:65536 >> gpurun_out/ab_pack.log 2>&1
for L in $D scripts/lib_pack.so; do echo "# $L"; HQC_LIB=$L timeout 300 python scripts/time_encrypt.py; done >> gpurun_out/ab_pack.log 2>&1
HQC_DEC_KERNEL=11 timeout 300 python scripts/time_kind.py 5:16384,5:20000 > gpurun_out/x5_small.log 2>&1
timeout 300 python scripts/time_kind.py 5:16384,5:16281,5:20000,5:65536 >> gpurun_out/x5_small.log 2>&1
