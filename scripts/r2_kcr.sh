# Round-2: k_out_cr (cell rows) parity + A/B against k_out (explicit) on C4.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "layouts_are_bitwise or concurrent_coarse or full_size_against_reference" > gpurun_out/r2e_parity.log 2>&1; echo "parity rc=$?"; tail -5 gpurun_out/r2e_parity.log
SWEEP_PROF=2 timeout 900 python scripts/sweep_env.py c4 "MSWM_KOUT=explicit" "MSWM_KOUT=cellrow" "MSWM_KOUT=explicit" "MSWM_KOUT=cellrow" > gpurun_out/r2e_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2e_sweep.log
for v in 5 8 4; do
MSWM_CUDA_LIB=paper_2106_07154_b200/_lib_ab/kcr$v.so SWEEP_PROF=2 timeout 600 python scripts/sweep_env.py c4 "MSWM_KOUT=cellrow" > gpurun_out/r2e_sweep_kcr$v.log 2>&1; echo "kcr$v rc=$?"; tail -1 gpurun_out/r2e_sweep_kcr$v.log
done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-rk4"
timeout 600 $B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_out_cr$" -c 1 -f -o gpurun_out/r2e_cr $B > gpurun_out/r2e_ncu_cr.log 2>&1; echo "ncu cr rc=$?"
MSWM_KOUT=explicit MSWM_HALO_DRYRUN=1 timeout 900 python scripts/rank_timing.py c4 8 10 > gpurun_out/r2e_rank_c4_8.json 2> gpurun_out/r2e_rank_c4_8.err; echo "rank timing rc=$?"; tail -3 gpurun_out/r2e_rank_c4_8.err; cut -c1-800 gpurun_out/r2e_rank_c4_8.json
