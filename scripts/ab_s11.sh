mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "fused_bc or optional or stencil" > gpurun_out/s11_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s11_pytest.log
SWEEP_STEPS=20 timeout 900 python scripts/sweep_env.py c4 "MSWM_BC=0" "MSWM_BC=1" "MSWM_BC=1 MSWM_BC_CELLS=128" "MSWM_BC=1 MSWM_BC_CELLS=512" "MSWM_BC=1 MSWM_BC_CELLS=1024" "MSWM_BC=0" "MSWM_BC=1" 2>&1 | tail -7 | cut -c1-130
timeout 900 python bench.py --config c5 --steps 20 > gpurun_out/s11_bench_c5.json 2> gpurun_out/s11_bench_c5.err; echo "bench c5 rc=$?"; tail -c 400 gpurun_out/s11_bench_c5.json
