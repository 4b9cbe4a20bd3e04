# session 5: state after the Omega truncation (RS_OMEGA_TERMS) — full GPU tests, smoke, bench, torchrun N=1, reference arm,
# ncu --set full of the default fused kernels, launch list of a short bench run
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_s5.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_s5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s5.log 2>&1; echo "exit $?" >> gpurun_out/smoke_s5.log
timeout 900 python bench.py > gpurun_out/bench_s5.log 2>&1
timeout 900 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/bench_torchrun_s5.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_s5.log 2>&1
run() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 300 "$@" > gpurun_out/s5_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/s5_$name "$@" > gpurun_out/s5_ncu_$name.log 2>&1
  echo "$name exit $?" >> gpurun_out/s5_status.log
}
run fused_L3 k_decrypt python scripts/prof_kernels.py --level 3 --batch 65536 --only fused --iters 2
run fused_L1 k_decrypt python scripts/prof_kernels.py --level 1 --batch 65536 --only fused --iters 2
run fused_L5 k_decrypt_s12c python scripts/prof_kernels.py --level 5 --batch 262144 --only fused --iters 2
run fused_L1_1024 k_decrypt python scripts/prof_kernels.py --level 1 --batch 1024 --only fused --iters 2
CMD="python bench.py --steps 5 --warmup 3 --no-configs --no-levels --no-variants --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/s5_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5_launches.csv $CMD > gpurun_out/s5_ncu_launches.log 2>&1
echo "launches exit $?" >> gpurun_out/s5_status.log
