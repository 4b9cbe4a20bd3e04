cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in scripts/libx_*.so; do echo "== $f" >> gpurun_out/exp.log; timeout 300 python scripts/par_lib.py $f >> gpurun_out/exp.log 2>&1; done
for r in 1 2; do for f in scripts/libx_*.so; do timeout 150 python scripts/time_lib.py $f 1,3,5 >> gpurun_out/exp.log 2>&1; done; done
