# fused-kernel time vs batch size (amortisation of the per-CTA RS tail), all levels; + quick parity
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not scaling_config and not round_trip_at_scale" > gpurun_out/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.log
for L in 1 3 5; do for B in 65536 131072 262144 524288; do
  echo "L$L B$B $(timeout 120 python scripts/prof_kernels.py --level $L --only fused --iters 10 --batch $B)" >> gpurun_out/batch.log
done; done
