# fused-kernel time vs start stagger (HQC_STAGGER_CYC), all levels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in 3 1 5; do for S in 0 20000 50000 100000 200000; do
  echo "L$L S$S $(HQC_STAGGER_CYC=$S timeout 120 python scripts/prof_kernels.py --level $L --only fused --iters 20)" >> gpurun_out/stagger.log
done; done
