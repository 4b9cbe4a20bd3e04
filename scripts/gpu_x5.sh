cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in 1 5 10 11; do HQC_DEC_KERNEL=$k timeout 300 python scripts/time_kind.py 5:16384,5:32768,5:65536,5:98304,5:131072,5:262144; done > gpurun_out/sweep_x5.log 2>&1
for k in 6 8 10 11; do HQC_DEC_KERNEL=$k timeout 300 python scripts/time_kind.py 1:65536,1:262144,3:65536,3:262144; done >> gpurun_out/sweep_x5.log 2>&1
for L in scripts/lib_u2.so paper_2512_12904_b200/libhqcgpu.so; do echo "# $L"; HQC_LIB=$L timeout 300 python scripts/time_encrypt.py; done > gpurun_out/enc_new.log 2>&1
