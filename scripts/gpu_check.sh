# GPU check of HEAD on one B200 (run under gpurun): the GPU suite (timed), smoke(), the default
# bench line and the per-rank timing of the 8-way C4 partition.  Outputs gpurun_out/<tag>_*.
#   bash scripts/gpu_check.sh <tag>
set -u
tag=${1:-check}
mkdir -p gpurun_out
t0=$(date +%s)
timeout 1500 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$? in $(( $(date +%s) - t0 )) s"; tail -32 gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/${tag}_bench_c4.json
MSWM_HALO_DRYRUN=1 timeout 900 python scripts/rank_timing.py c4 8 10 > gpurun_out/${tag}_rank_c4_8.json 2> gpurun_out/${tag}_rank_c4_8.err; echo "rank timing rc=$?"; tail -2 gpurun_out/${tag}_rank_c4_8.err
