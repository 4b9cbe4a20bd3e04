cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for K in 1 6; do
  CMD="python scripts/prof_kernels.py --level 5 --batch 65536 --only fused --iters 2"
  HQC_DEC_KERNEL=$K timeout 300 $CMD > gpurun_out/prof_wd5_plain_K$K.log 2>&1 && \
  HQC_DEC_KERNEL=$K timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decrypt -s 3 -c 1 -o gpurun_out/prof_wd5_K$K $CMD > gpurun_out/ncu_wd5_K$K.log 2>&1
  echo "K$K exit $?" >> gpurun_out/ncu_wd5_status.log
done
