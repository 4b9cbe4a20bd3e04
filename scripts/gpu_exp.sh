cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for f in scripts/libx_*.so; do timeout 150 python scripts/time_lib.py $f 3 >> gpurun_out/exp.log 2>&1; timeout 150 python scripts/time_lib.py $f 3 262144 >> gpurun_out/exp.log 2>&1; done; done
