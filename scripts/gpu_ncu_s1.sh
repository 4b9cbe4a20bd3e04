# ncu --set full of the standalone product's default kernels (k_stage1 at HQC-1/3, k_stage1p at HQC-5),
# v = NULL, 65,536 products, one launch each after warm-up
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in 1 3 5; do
  CMD="python scripts/prof_kernels.py --level $L --only s1n --iters 2"
  timeout 300 $CMD > gpurun_out/prof_s1n_plain_L$L.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage1 -s 3 -c 1 -o gpurun_out/prof_s1n_L$L $CMD > gpurun_out/ncu_s1n_L$L.log 2>&1
  echo "L$L exit $?" >> gpurun_out/ncu_s1n_status.log
done
