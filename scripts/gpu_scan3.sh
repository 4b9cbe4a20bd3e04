cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
HQC_DEC_KERNEL=8 timeout 600 python scripts/time_kind.py 3:45000,3:49152,3:57344,3:65536,3:73728,3:81920,3:98304,3:131072,3:196608,3:262144,3:393216,3:524288 > gpurun_out/scan3.log 2>&1
HQC_DEC_KERNEL=6 timeout 600 python scripts/time_kind.py 1:49152,1:57344,1:65536,1:73728,1:81920,1:98304,1:131072 >> gpurun_out/scan3.log 2>&1
