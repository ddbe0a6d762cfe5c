mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s9_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s9_pytest.log
for v in head pk3k0 pk3k1 pk2k0 head pk3k0; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=20 timeout 300 python scripts/sweep_env.py c4 "MSWM_ST16=1" "MSWM_ST16=1" 2>&1 | tail -2 | cut -c1-120
done
