# Round-2: k_out_rw vs k_out A/B sweep on C4, then one ncu full capture of each output kernel.
set -u
mkdir -p gpurun_out
SWEEP_PROF=2 timeout 900 python scripts/sweep_env.py c4 "MSWM_KOUT=explicit" "MSWM_RW_CELLS=128" "MSWM_RW_CELLS=64" \
  "MSWM_RW_CELLS=256 MSWM_RW_STAGE_KB=64" "MSWM_RW_CELLS=32 MSWM_RW_STAGE_KB=12" "MSWM_KOUT=explicit" > gpurun_out/r2c_sweep.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/r2c_sweep.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-rk4"
timeout 600 $B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_out_rw$" -s 2 -c 1 -f -o gpurun_out/r2c_rw $B > gpurun_out/r2c_ncu_rw.log 2>&1; echo "ncu rw rc=$?"
MSWM_KOUT=explicit timeout 600 $B > /dev/null 2>&1 && MSWM_KOUT=explicit timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_out$" -s 2 -c 1 -f -o gpurun_out/r2c_ex $B > gpurun_out/r2c_ncu_ex.log 2>&1; echo "ncu ex rc=$?"
