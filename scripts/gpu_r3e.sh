for rep in 1 2; do
HQC_DEC_KERNEL=1 python scripts/time_kind.py 5:131072,5:4194304
HQC_DEC_KERNEL=10 python scripts/time_kind.py 5:131072,5:98304
for sp in 262144 1048576 0; do HQC_DEC_KERNEL=10 HQC_DEC_SPLIT=$sp python scripts/time_kind.py 5:4194304; done
done
