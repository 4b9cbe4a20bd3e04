# full GPU check: all gpu tests, smoke, bench per level (+ torchrun world 1), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for L in 1 5; do timeout 600 python bench.py --level $L --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1; done
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_torchrun.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
