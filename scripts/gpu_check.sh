# quick: GPU parity suite (minus the slow full-size cases) + fused-kernel timings for all levels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "not full_size and not scaling_config and not round_trip_at_scale" > gpurun_out/pytest_quick.log 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.log
for L in 1 3 5; do timeout 120 python scripts/prof_kernels.py --level $L --only fused --iters 20 >> gpurun_out/timing.log 2>&1; done
