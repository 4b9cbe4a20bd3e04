cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python scripts/prof_kem.py --levels 3 --iters 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encrypt2 -s 1 -c 1 -o gpurun_out/prof_enc2_L3 $CMD > gpurun_out/ncu_enc2.log 2>&1
HQC_ENC_KERNEL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_encrypt -s 1 -c 1 -o gpurun_out/prof_enc1_L3 $CMD > gpurun_out/ncu_enc1.log 2>&1
