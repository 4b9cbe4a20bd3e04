cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or two_launch" > gpurun_out/pytest_k4c.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k4c.log
for rep in 1 2; do
for k in 10 11; do HQC_DEC_KERNEL=$k timeout 300 python scripts/time_kind.py 5:262144,5:1048576,5:131072,3:65536,1:65536; done
done > gpurun_out/ab_k4c.log 2>&1
