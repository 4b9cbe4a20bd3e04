cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for f in scripts/libx_*.so; do echo "$f $(timeout 200 python scripts/time_kem_lib.py $f 3,5 2>&1 | tail -1)" >> gpurun_out/exp.log; done; done
echo "old $(HQC_ENC_KERNEL=1 timeout 200 python scripts/time_kem_lib.py scripts/libx_e2_base.so 3,5 2>&1 | tail -1)" >> gpurun_out/exp.log
