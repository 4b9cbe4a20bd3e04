# new KEM keygen tests + ncu --set full of the standalone product kernel (k_stage1) at HQC-3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kem.py -q -x > gpurun_out/pytest_kem.log 2>&1; echo "exit $?" >> gpurun_out/pytest_kem.log
L=${L:-3}
CMD="python scripts/prof_kernels.py --level $L --only s1 --iters 2"
timeout 300 $CMD > gpurun_out/prof_s1_plain_L$L.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage1 -s 3 -c 1 -o gpurun_out/prof_s1_L$L $CMD > gpurun_out/ncu_s1_L$L.log 2>&1
echo "exit $?" >> gpurun_out/ncu_s1_L$L.log
