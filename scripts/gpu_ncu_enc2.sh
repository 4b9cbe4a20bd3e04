cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for L in 1 3; do
  CMD="python scripts/time_encrypt.py $L"
  timeout 300 $CMD > gpurun_out/enc_plain_L$L.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_encrypt2 -s 1 -c 1 -o gpurun_out/prof_enc2b_L$L $CMD > gpurun_out/ncu_enc2b_L$L.log 2>&1
  echo "L$L exit $?" >> gpurun_out/ncu_enc_status.log
done
