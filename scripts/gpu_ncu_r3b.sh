cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r3_*.ncu-rep
run() {  # name, kernel regex, command...
  local name=$1 rx=$2; shift 2
  timeout 300 "$@" > gpurun_out/r3_plain_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 -o gpurun_out/r3_$name "$@" > gpurun_out/r3_ncu_$name.log 2>&1
  echo "$name exit $?" >> gpurun_out/r3_status.log
}
run x12_L5 k_decrypt_s12 python scripts/time_kind.py 5:262144
