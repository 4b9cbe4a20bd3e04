cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for K in 1 2; do echo "K$K $(HQC_DEC_KERNEL=$K timeout 150 python scripts/time_lib.py scripts/libx_sw5.so 5 262144)" >> gpurun_out/exp.log; done; done
HQC_DEC_KERNEL=2 timeout 300 python scripts/par_lib.py scripts/libx_sw5.so >> gpurun_out/exp.log 2>&1
