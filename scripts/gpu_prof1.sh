cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in 1 3 5; do timeout 300 python scripts/prof_kernels.py --level $L > gpurun_out/prof_split_L$L.log 2>&1; done
CMD="python scripts/prof_kernels.py --level 3 --only fused --iters 2"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decrypt -s 3 -c 1 -o gpurun_out/prof_fused_L3 $CMD > gpurun_out/ncu_fused.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_fused.log
