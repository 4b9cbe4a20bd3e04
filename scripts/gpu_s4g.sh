# session 4: compute-sanitizer on the warp-decoder kernels after riBM / tournament (sb = 5, sp = 7)
# (on this pool the sanitizer is closed: every run printed "compute-sanitizer is closed on this pool" and exit 86)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for TOOL in memcheck racecheck synccheck; do for K in 5 7; do
HQC_DEC_KERNEL=$K SAN_DEC_ONLY=1 SAN_B=40 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 20 python scripts/sanitize_run.py > gpurun_out/san4_${TOOL}_k$K.log 2>&1; echo "exit $?" >> gpurun_out/san4_${TOOL}_k$K.log
done; done
