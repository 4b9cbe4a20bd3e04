# round-2 ncu evidence of the default kernels (one capture each, after the same command ran plain)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 300 "$@" > gpurun_out/final_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/final_$name "$@" > gpurun_out/final_ncu_$name.log 2>&1
  echo "$name exit $?" >> gpurun_out/final_status.log
}
run fused_L1 k_decrypt python scripts/prof_kernels.py --level 1 --batch 65536 --only fused --iters 2
run fused_L3 k_decrypt python scripts/prof_kernels.py --level 3 --batch 65536 --only fused --iters 2
run fused_L5 k_decrypt python scripts/prof_kernels.py --level 5 --batch 262144 --only fused --iters 2
run fused_L1_1024 k_decrypt python scripts/prof_kernels.py --level 1 --batch 1024 --only fused --iters 2
