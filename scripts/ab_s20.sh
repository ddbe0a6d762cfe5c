mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s20_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/s20_pytest.log
for v in head2 split; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=30 timeout 900 python scripts/sweep_env.py c4 "MSWM_FORK=1" "MSWM_FORK=1 MSWM_FORK_CTAS=7" "MSWM_FORK=1 MSWM_FORK_CTAS=5" "MSWM_FORK=1" 2>&1 | tail -4 | cut -c1-120
done
