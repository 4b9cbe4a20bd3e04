# ncu --set full captures of the KEM kernels (k_encrypt compare mode, k_kem_kdf, k_kem_coins) at HQC-3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/prof_kem.py --levels 3 --iters 1"
timeout 300 $CMD > gpurun_out/kem_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for K in k_encrypt k_kem_kdf k_kem_coins; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/kem_$K $CMD > gpurun_out/ncu_kem_$K.log 2>&1
  echo "$K exit $?"
done
