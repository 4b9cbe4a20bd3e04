cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q > gpurun_out/pytest_split2.log 2>&1; echo "exit $?" >> gpurun_out/pytest_split2.log
timeout 600 python scripts/time_kind.py 1:65536,1:73728,1:81920,1:131072,1:4194304,3:65536,3:98304,3:524288,3:1048576,3:4194304 > gpurun_out/split2.log 2>&1
HQC_DEC_SPLIT=0 timeout 600 python scripts/time_kind.py 1:73728,1:81920 >> gpurun_out/split2.log 2>&1
HQC_DEC_KERNEL=8 timeout 600 python scripts/time_kind.py 3:1048576 >> gpurun_out/split2.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_split2.log 2>&1
