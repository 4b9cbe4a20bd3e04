cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
D=paper_2512_12904_b200/libhqcgpu.so
for L in scripts/lib_u2.so scripts/lib_u3.so scripts/lib_u2.so scripts/lib_u3.so; do echo "# $L"; HQC_LIB=$L timeout 300 python scripts/time_encrypt.py; done > gpurun_out/ab_unroll_enc.log 2>&1
timeout 600 python scripts/exp_lib_ab.py scripts/lib_u2.so $D 5:262144,3:65536,1:65536,1:1024 > gpurun_out/ab_unroll_new.log 2>&1
timeout 600 python scripts/exp_s1_ab.py scripts/lib_u3.so $D s1:5:65536,s1:3:65536,s1:1:65536 >> gpurun_out/ab_unroll_new.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_unroll.log 2>&1; echo "exit $?" >> gpurun_out/pytest_unroll.log
