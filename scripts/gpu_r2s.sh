# round 2 (session 3): tests, bench and ncu of the segmented-layout defaults and K4c
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_s.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_s.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s.log 2>&1; echo "exit $?" >> gpurun_out/smoke_s.log
timeout 900 python bench.py > gpurun_out/bench_s.log 2>&1
run() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 300 "$@" > gpurun_out/s_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/s_$name "$@" > gpurun_out/s_ncu_$name.log 2>&1
  echo "$name exit $?" >> gpurun_out/s_status.log
}
run fused_L3 k_decrypt python scripts/prof_kernels.py --level 3 --batch 65536 --only fused --iters 2
run fused_L1 k_decrypt python scripts/prof_kernels.py --level 1 --batch 65536 --only fused --iters 2
run fused_L5 k_decrypt_s12c python scripts/prof_kernels.py --level 5 --batch 262144 --only fused --iters 2
run s1n_L1 k_stage1 python scripts/prof_kernels.py --level 1 --only s1n --iters 2
run s1n_L3 k_stage1 python scripts/prof_kernels.py --level 3 --only s1n --iters 2
CMD="python bench.py --steps 5 --warmup 3 --no-configs --no-levels --no-variants --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/s_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s_launches.csv $CMD > gpurun_out/s_ncu_launches.log 2>&1
echo "launches exit $?" >> gpurun_out/s_status.log
