# Round-2 check: GPU suite (timed), smoke, default bench line, per-rank timing of the 8-way C4 partition.
set -u
mkdir -p gpurun_out
nproc > gpurun_out/r2f_host.txt
/usr/bin/time -v timeout 1500 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/r2f_pytest.log 2> gpurun_out/r2f_pytest.time; echo "pytest rc=$?"; tail -28 gpurun_out/r2f_pytest.log; grep "Elapsed\|Maximum resident" gpurun_out/r2f_pytest.time
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2f_smoke.log
timeout 900 python bench.py > gpurun_out/r2f_bench_c4.json 2> gpurun_out/r2f_bench_c4.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/r2f_bench_c4.json
MSWM_HALO_DRYRUN=1 timeout 900 python scripts/rank_timing.py c4 8 10 > gpurun_out/r2f_rank_c4_8.json 2> gpurun_out/r2f_rank_c4_8.err; echo "rank timing rc=$?"; tail -2 gpurun_out/r2f_rank_c4_8.err
MSWM_HALO_DRYRUN=1 MSWM_OVERLAP=0 timeout 900 python scripts/rank_timing.py c4 8 10 > gpurun_out/r2f_rank_c4_8_nooverlap.json 2> gpurun_out/r2f_rank_c4_8_nooverlap.err; echo "rank timing (no overlap) rc=$?"
