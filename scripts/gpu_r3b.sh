C=5:262144
for rep in 1 2; do
HQC_DEC_KERNEL=1 python scripts/time_kind.py $C
for s in 0 1000 3000 6000 12000; do HQC_DEC_KERNEL=10 HQC_S12_STAGGER=$s python scripts/time_kind.py $C; done
HQC_DEC_KERNEL=10 HQC_DEC_SPLIT=0 python scripts/time_kind.py 5:1048576
HQC_DEC_KERNEL=1 python scripts/time_kind.py 5:1048576
done
