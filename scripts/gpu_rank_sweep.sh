# Per-rank timing (scripts/rank_timing.py, dry run: no kernels wait on one another) of the C4
# partition at 2 / 4 / 8 ranks and of C5 at 8 ranks, for the latency model (scripts/latency_model.py).
set -u
mkdir -p gpurun_out
for n in 2 4 8; do
  MSWM_HALO_DRYRUN=1 timeout 900 python scripts/rank_timing.py c4 $n 10 > gpurun_out/rs_c4_$n.json 2> gpurun_out/rs_c4_$n.err; echo "c4 x$n rc=$?"
done
MSWM_HALO_DRYRUN=1 timeout 2400 python scripts/rank_timing.py c5 8 5 > gpurun_out/rs_c5_8.json 2> gpurun_out/rs_c5_8.err; echo "c5 x8 rc=$?"; tail -3 gpurun_out/rs_c5_8.err
