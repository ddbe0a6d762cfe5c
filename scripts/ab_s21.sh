mkdir -p gpurun_out
SWEEP_STEPS=30 timeout 1200 python scripts/sweep_env.py c4 "MSWM_KERNELS=explicit" "MSWM_KERNELS=auto" "MSWM_KERNELS=auto MSWM_TILE_CELLS=128" "MSWM_KERNELS=auto MSWM_TILE_CELLS=64" "MSWM_KERNELS=auto MSWM_FORK_CTAS=7" "MSWM_KERNELS=explicit" 2>&1 | tail -6 | cut -c1-120
