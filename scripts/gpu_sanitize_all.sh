# every kernel on small batches, checked against the oracle (scripts/sanitize_run.py); compute-sanitizer
# itself is not available on this GPU pool, so the run is the plain one
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "exit $?" >> gpurun_out/san_plain.log
