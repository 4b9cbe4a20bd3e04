cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_t.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_t.log 2>&1; echo "exit $?" >> gpurun_out/smoke_t.log
timeout 900 python bench.py > gpurun_out/bench_t.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_t.log 2>&1
timeout 600 python scripts/time_stages.py > gpurun_out/time_stages_t.log 2>&1
