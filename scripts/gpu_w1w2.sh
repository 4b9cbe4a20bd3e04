cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
HQC_DEC_KERNEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "decrypt" > gpurun_out/pytest_w1.log 2>&1; echo "w1 pytest exit $?" >> gpurun_out/pytest_w1.log
for K in 1 2; do for L in 1 3 5; do HQC_DEC_KERNEL=$K timeout 300 python scripts/prof_kernels.py --level $L --only fused > gpurun_out/w${K}_L$L.log 2>&1; done; done
