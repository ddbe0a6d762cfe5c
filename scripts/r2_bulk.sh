# Round-2: k_out_bulk (bulk-copy table stream) parity + A/B on C4.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "concurrent or layouts" > gpurun_out/r2b2_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2b2_parity.log
SWEEP_PROF=2 timeout 900 python scripts/sweep_env.py c4 "MSWM_BULK=0" "MSWM_BULK=1" "MSWM_BULK=0" "MSWM_BULK=1" > gpurun_out/r2b2_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2b2_sweep.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-rk4"
MSWM_BULK=1 timeout 600 $B > /dev/null 2>&1 && MSWM_BULK=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_out_bulk$" -c 1 -f -o gpurun_out/r2b2_bulk $B > gpurun_out/r2b2_ncu.log 2>&1; echo "ncu rc=$?"
