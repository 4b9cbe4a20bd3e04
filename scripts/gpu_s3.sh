cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
timeout 600 python scripts/exp_lib_ab.py $D scripts/lib_s3m4.so 5:262144,5:65536 > gpurun_out/ab_s3.log 2>&1
for L in $D scripts/lib_s3m4.so; do echo "# $L"; HQC_LIB=$L timeout 300 python scripts/time_stages.py 5:262144 3:65536 1:65536; done >> gpurun_out/ab_s3.log 2>&1
