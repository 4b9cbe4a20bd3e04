cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in scripts/libx_*.so; do echo "== $f" >> gpurun_out/exp.log; timeout 300 python scripts/par_lib.py $f >> gpurun_out/exp.log 2>&1; done
for r in 1 2; do for f in scripts/libx_*.so paper_2512_12904_b200/libhqcgpu.so; do timeout 150 python scripts/time_lib.py $f 3 >> gpurun_out/exp.log 2>&1; done; done
