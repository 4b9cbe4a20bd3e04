# compute-sanitizer, ONE tool per call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck|initcheck
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/sanitize_run.py > gpurun_out/san_plain.log 2>&1 && \
for K in 1 2 3; do HQC_DEC_KERNEL=$K SAN_B=40 timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san_${TOOL}_k$K.log 2>&1; echo "exit $?" >> gpurun_out/san_${TOOL}_k$K.log; done
