# syndrome-method parity + timing + ncu metrics; the configs[4] full-size tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "syndromes" > gpurun_out/pytest_syn.log 2>&1; echo "exit $?" >> gpurun_out/pytest_syn.log
timeout 300 python scripts/prof_syndromes.py > gpurun_out/syn_timing.log 2>&1
for M in linear nibble logexp; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_syndromes -s 2 -c 1 -o gpurun_out/prof_syn_${M}_L3 python scripts/prof_syndromes.py --levels 3 --methods $M --iters 1 > gpurun_out/ncu_syn_$M.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_encrypt.py -q -x -k "scaling_config" --durations=5 > gpurun_out/pytest_scaling.log 2>&1; echo "exit $?" >> gpurun_out/pytest_scaling.log
