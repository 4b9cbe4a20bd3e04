# session 4: phase counters of k_decrypt_sp (warp pair) vs k_decrypt_sb at 512 / 1,024
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/exp_sb_phases.py run > gpurun_out/phases_sb_s4.log 2>&1
HQC_DEC_KERNEL=7 timeout 300 python scripts/exp_sb_phases.py run > gpurun_out/phases_sp_s4.log 2>&1
