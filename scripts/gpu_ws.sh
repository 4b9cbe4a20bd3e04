cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variants" > gpurun_out/pytest_ws.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ws.log
for K in 2 3; do for L in 1 3 5; do HQC_DEC_KERNEL=$K timeout 300 python scripts/prof_kernels.py --level $L --only fused > gpurun_out/w${K}_L$L.log 2>&1; done; done
