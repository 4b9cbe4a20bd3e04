for g in 0 8 7; do for w in 4 1 2; do
HQC_S1_G=$g HQC_S3_WARPS=$w python scripts/exp_overlap.py 5 1048576 131072
done; done
