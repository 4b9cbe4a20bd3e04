cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host" > gpurun_out/pytest_ct.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ct.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-levels > gpurun_out/bench_ct.log 2>&1; echo "exit $?" >> gpurun_out/bench_ct.log
