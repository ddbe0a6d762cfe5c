mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s7_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s7_pytest.log
SWEEP_STEPS=20 timeout 600 python scripts/sweep_env.py c4 "MSWM_IDX16=1" "MSWM_IDX16=0" "MSWM_IDX16=1" "MSWM_IDX16=0" 2>&1 | tail -5 | cut -c1-120
