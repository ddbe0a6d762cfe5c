mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "compressed or c2_full or layouts or optional or golden" > gpurun_out/s8_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s8_pytest.log
SWEEP_STEPS=20 timeout 900 python scripts/sweep_env.py c4 "MSWM_IDX16=31" "MSWM_IDX16=0" "MSWM_IDX16=24" "MSWM_IDX16=7" "MSWM_IDX16=1" "MSWM_IDX16=6" "MSWM_IDX16=31" "MSWM_IDX16=0" 2>&1 | tail -8 | cut -c1-120
