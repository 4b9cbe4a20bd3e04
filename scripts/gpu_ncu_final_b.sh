# round-2 ncu evidence of the default kernels (one capture each, after the same command ran plain)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 300 "$@" > gpurun_out/final_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/final_$name "$@" > gpurun_out/final_ncu_$name.log 2>&1
  echo "$name exit $?" >> gpurun_out/final_status.log
}
run s1n_L1 k_stage1 python scripts/prof_kernels.py --level 1 --only s1n --iters 2
run s1n_L3 k_stage1 python scripts/prof_kernels.py --level 3 --only s1n --iters 2
run s1n_L5 k_stage1 python scripts/prof_kernels.py --level 5 --only s1n --iters 2
# launch list of a short bench run (headline only)
CMD="python bench.py --steps 5 --warmup 3 --no-configs --no-levels --no-variants --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/final_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_ncu_launches.log 2>&1
echo "launches exit $?" >> gpurun_out/final_status.log
