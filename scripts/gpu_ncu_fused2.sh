# ncu --set full of the fused decrypt defaults: HQC-1 (k_decrypt_w1, 65,536), HQC-3 (k_decrypt_sb, 65,536),
# HQC-5 (k_decrypt_w1, 262,144), and configs[0] (k_decrypt_sb, HQC-1, 1,024)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in "1 65536" "3 65536" "5 262144" "1 1024"; do
  set -- $spec
  CMD="python scripts/prof_kernels.py --level $1 --batch $2 --only fused --iters 2"
  timeout 300 $CMD > gpurun_out/prof_fused_plain_L$1_B$2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decrypt -s 3 -c 1 -o gpurun_out/prof_fused_L$1_B$2 $CMD > gpurun_out/ncu_fused_L$1_B$2.log 2>&1
  echo "L$1 B$2 exit $?" >> gpurun_out/ncu_fused_status.log
done
