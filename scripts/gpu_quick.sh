# quick GPU check: parity tests (fast subset) + per-kernel timings for all levels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for L in 1 3 5; do timeout 300 python scripts/prof_kernels.py --level $L > gpurun_out/prof_split_L$L.log 2>&1; done
