# ncu evidence: launch list of the bench command + one full capture of the fused kernel per level
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BCMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 $BCMD > gpurun_out/ncu_bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launches.log 2>&1
for L in 1 3 5; do
  CMD="python scripts/prof_kernels.py --level $L --only fused --iters 2"
  timeout 300 $CMD > gpurun_out/prof_plain_L$L.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decrypt -s 3 -c 1 -o gpurun_out/prof_fused_L$L $CMD > gpurun_out/ncu_fused_L$L.log 2>&1
done
