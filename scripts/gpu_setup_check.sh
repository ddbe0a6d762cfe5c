# Host-parallel table build on one B200 (under gpurun): parity subset incl. the full-size comparisons,
# the bench line (setup times), and a sweep of the concurrent coarse stage's CTAs per SM.
set -u
tag=${1:-setup}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_dropin.py tests/test_horizon.py -q -m gpu -x -k "not c5" --durations=8 \
  > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/${tag}_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/${tag}_bench_c4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['roofline']['ms'],d['roofline'].get('ms_min'),d['roofline'].get('ms_max'),d['setup'])"
SWEEP_STEPS=20 timeout 900 python scripts/sweep_env.py c4 "MSWM_FORK_CTAS=6" "MSWM_FORK_CTAS=5" "MSWM_FORK_CTAS=7" "MSWM_FORK_CTAS=6" "MSWM_FORK_CTAS=5" "MSWM_FORK_CTAS=7" \
  > gpurun_out/${tag}_fork_sweep.log 2>&1; echo "sweep rc=$?"; cut -c1-140 gpurun_out/${tag}_fork_sweep.log | tail -6
