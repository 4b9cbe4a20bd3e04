cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HQC_DEC_KERNEL=8 timeout 600 python scripts/time_kind.py 3:131072,3:262144,3:524288,3:1048576,3:4194304 > gpurun_out/sweep_x3.log 2>&1
for sp in 0 262144 1048576; do HQC_DEC_KERNEL=10 HQC_DEC_SPLIT=$sp timeout 600 python scripts/time_kind.py 3:131072,3:262144,3:524288,3:1048576,3:4194304; done >> gpurun_out/sweep_x3.log 2>&1
for sp in 0 262144 1048576; do HQC_DEC_KERNEL=11 HQC_DEC_SPLIT=$sp timeout 600 python scripts/time_kind.py 5:1048576,5:4194304; done >> gpurun_out/sweep_x3.log 2>&1
