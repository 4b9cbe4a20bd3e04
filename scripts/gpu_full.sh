# one GPU call: smoke, parity suite, bench (default + per level), reference arm, launch list, ncu --set full of the fused kernel per level
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | head -20; nvidia-smi; free -g) > gpurun_out/sys.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
[ -n "$NO_NCU" ] && exit 0
BCMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launches.log 2>&1
for L in 1 3 5; do
  CMD="python scripts/prof_kernels.py --level $L --only fused --iters 2"
  timeout 300 $CMD > gpurun_out/prof_plain_L$L.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decrypt -s 3 -c 1 -o gpurun_out/prof_fused_L$L $CMD > gpurun_out/ncu_fused_L$L.log 2>&1
done
for L in 3 5; do  # the opt-in tensor-memory standalone product (k_stage1t, HQC_S1_KERNEL=3)
  HQC_S1_KERNEL=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage1t -s 3 -c 1 -f -o gpurun_out/prof_s1t_L$L python scripts/time_s1_lib.py paper_2512_12904_b200/libhqcgpu.so $L > gpurun_out/ncu_s1t_L$L.log 2>&1
done
