# Round-2 check: GPU suite (timed), smoke, default bench line, per-rank timing of the 8-way C4 partition.
set -u
mkdir -p gpurun_out
t0=$(date +%s)
timeout 1500 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$? in $(( $(date +%s) - t0 )) s"; tail -32 gpurun_out/r2g_pytest.log
timeout 900 python bench.py > gpurun_out/r2g_bench_c4.json 2> gpurun_out/r2g_bench_c4.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r2g_bench_c4.json
MSWM_HALO_DRYRUN=1 timeout 900 python scripts/rank_timing.py c4 8 10 > gpurun_out/r2g_rank_c4_8.json 2> gpurun_out/r2g_rank_c4_8.err; echo "rank timing rc=$?"; tail -2 gpurun_out/r2g_rank_c4_8.err
