cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | head -20; nvidia-smi; free -g) > gpurun_out/sys.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for L in 1 3 5; do timeout 600 python bench.py --steps 10 --warmup 3 --level $L --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
