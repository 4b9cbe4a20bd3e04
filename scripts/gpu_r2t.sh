# the N = 2 bench path (torchrun, two ranks) on ONE GPU with gloo collectives: a logic check, not a measurement
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HQC_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-variants --config5-total 1048576 > gpurun_out/bench_n2_gloo.log 2>&1
echo "exit $?" >> gpurun_out/bench_n2_gloo.log
