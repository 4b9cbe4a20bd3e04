cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_split.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_split.log
timeout 600 python scripts/time_kind.py 1:65536,1:73728,1:81920,1:131072,1:1048576,1:4194304,3:65536,3:81920,3:98304,3:262144,3:4194304 > gpurun_out/split_new.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_split.log 2>&1
