cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 300 "$@" > gpurun_out/x_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/x_$name "$@" > gpurun_out/x_ncu_$name.log 2>&1
  echo "$name exit $?" >> gpurun_out/x_status.log
}
run sb_L1_1024 k_decrypt_sb python scripts/prof_kernels.py --level 1 --batch 1024 --only fused --iters 2
run wc_L3_262144 k_decrypt_wc python scripts/prof_kernels.py --level 3 --batch 262144 --only fused --iters 2
run wl_L3_4M k_decrypt_wl python scripts/prof_kernels.py --level 3 --batch 4194304 --only fused --iters 1
