mkdir -p gpurun_out
for v in head2 hint; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=30 timeout 900 python scripts/sweep_env.py c4 "MSWM_L2HINT=00" "MSWM_L2HINT=01" "MSWM_L2HINT=20" "MSWM_L2HINT=21" "MSWM_L2HINT=00" 2>&1 | tail -5 | cut -c1-100
done
