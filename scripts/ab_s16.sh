mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s16_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/s16_pytest.log
SWEEP_STEPS=30 timeout 900 python scripts/sweep_env.py c4 "MSWM_FORK=0" "MSWM_FORK=1" "MSWM_FORK=0" "MSWM_FORK=1" 2>&1 | tail -4 | cut -c1-100
