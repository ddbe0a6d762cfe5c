mkdir -p gpurun_out
for v in head4 ka6 head4 ka6; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=30 timeout 600 python scripts/sweep_env.py c4 "MSWM_FORK=1" 2>&1 | tail -1 | cut -c1-100
done
