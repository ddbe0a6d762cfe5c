mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "concurrent or c2_full or golden" > gpurun_out/s18_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s18_pytest.log
SWEEP_STEPS=30 timeout 900 python scripts/sweep_env.py c4 "MSWM_FORK_CTAS=6" "MSWM_FORK_CTAS=6,6,8" "MSWM_FORK_CTAS=5,5,8" "MSWM_FORK_CTAS=6,6,7" "MSWM_FORK_CTAS=4,4,8" "MSWM_FORK_CTAS=7,7,8" "MSWM_FORK_CTAS=6" 2>&1 | tail -7 | cut -c1-110
