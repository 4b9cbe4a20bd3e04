cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for K in 2 3 1; do HQC_DEC_KERNEL=$K timeout 150 python scripts/time_lib.py paper_2512_12904_b200/libhqcgpu.so 1,3,5 >> gpurun_out/exp.log 2>&1; done; done
