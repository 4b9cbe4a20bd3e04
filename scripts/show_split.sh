tail -2 gpurun_out/pytest_gpu.log
for L in 1 3 5; do python -c "import json,sys; d=json.load(open('gpurun_out/prof_split_L$L.log')); print(d['level'], {k:(round(v['ms'],3), '%.3g'%v['decryptions_per_s']) for k,v in d.items() if isinstance(v,dict) and 'ms' in v})" 2>&1 | tail -1; done
