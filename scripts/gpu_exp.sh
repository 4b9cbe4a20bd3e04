cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 4096 8192 16384 32768; do echo "chunk $c $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-levels --e2e-steps 5 --e2e-chunk $c 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d["e2e"]))')" >> gpurun_out/exp.log; done
