cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/pytest_wc2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_wc2.log
for rep in 1 2; do
for k in 8 12; do HQC_DEC_KERNEL=$k timeout 300 python scripts/time_kind.py 3:65536,3:131072,3:262144,3:4194304; done
done > gpurun_out/ab_wc2.log 2>&1
