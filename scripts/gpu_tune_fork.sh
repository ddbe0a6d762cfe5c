# Fork CTA split sweep on C4 plus the drop-in / stencil tests and a bench line (tuning run).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -x -k "stencil or layouts or dropin or packed or stepper or concurrent" > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2k_tests.log
SWEEP_PROF=2 timeout 1200 python scripts/sweep_env.py c4 "MSWM_FORK_CTAS=6" "MSWM_FORK_CTAS=4" "MSWM_FORK_CTAS=5" "MSWM_FORK_CTAS=7" "MSWM_FORK_CTAS=8" "MSWM_FORK_CTAS=8,8,6" "MSWM_FORK_CTAS=6,6,4" "MSWM_FORK_CTAS=6" > gpurun_out/r2k_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2k_sweep.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2k_bench_c4.json 2> gpurun_out/r2k_bench_c4.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r2k_bench_c4.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms'], d['e2e_dropin_eval']['ms_per_coarse_step'], d['clocks'])"
