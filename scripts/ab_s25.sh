mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "not full_size" > gpurun_out/s25_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s25_pytest.log
for v in head5 member head5 member; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=30 timeout 600 python scripts/sweep_env.py c4 "MSWM_FORK=1" "MSWM_FORK=0" 2>&1 | tail -2 | cut -c1-100
done
