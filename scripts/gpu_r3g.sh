timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "variants and 11" 2>&1 | tail -2
for rep in 1 2; do
HQC_DEC_KERNEL=10 python scripts/time_kind.py 5:262144
for r in 1 2 3; do HQC_DEC_KERNEL=11 HQC_X_RM=$r timeout 120 python scripts/time_kind.py 5:262144; done
HQC_DEC_KERNEL=11 HQC_X_RM=2 HQC_S1_G=8 timeout 120 python scripts/time_kind.py 5:262144
done
for l in 1 3; do for k in 10 11; do HQC_DEC_KERNEL=$k timeout 120 python scripts/time_kind.py $l:65536; done; done
