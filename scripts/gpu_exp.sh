cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for r in 1 2; do for f in scripts/libx_*.so; do echo "$f $(timeout 200 python scripts/time_kem_lib.py $f 1,3,5 2>&1 | tail -1)" >> gpurun_out/exp.log; done; done
