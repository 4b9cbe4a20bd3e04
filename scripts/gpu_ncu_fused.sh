cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in 1 3 5; do
  CMD="python scripts/prof_kernels.py --level $L --only fused --iters 2"
  timeout 300 $CMD > gpurun_out/prof_plain_L$L.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decrypt -s 3 -c 1 -o gpurun_out/prof_fused_L$L $CMD > gpurun_out/ncu_fused_L$L.log 2>&1
done
