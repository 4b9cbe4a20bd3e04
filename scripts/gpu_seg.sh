cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_seg.log 2>&1; echo "exit $?" >> gpurun_out/pytest_seg.log
A=scripts/lib_seg0.so; B=paper_2512_12904_b200/libhqcgpu.so
timeout 600 python scripts/exp_lib_ab.py $A $B 1:65536,3:65536,5:262144,1:1024,3:1024,5:1024,3:16384 > gpurun_out/ab_seg_dec.log 2>&1
timeout 600 python scripts/exp_s1_ab.py $A $B s1:1:65536,s1:3:65536,s1:5:65536 > gpurun_out/ab_seg_s1.log 2>&1
for L in $A $B $A $B; do echo "# $L"; HQC_LIB=$L timeout 300 python scripts/time_encrypt.py; done > gpurun_out/ab_seg_enc.log 2>&1
