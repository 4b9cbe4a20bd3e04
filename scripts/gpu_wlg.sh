cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for g in 16 15 14 13 12; do HQC_WL_G=$g timeout 300 python scripts/time_kind.py 3:65536,3:57344,3:49152; done > gpurun_out/wlg.log 2>&1
