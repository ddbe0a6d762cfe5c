# Chunk schedules (MSWM_MIX / MSWM_MIX_WIN) on one B200 (under gpurun): parity of the schedules on the
# small GPU tests, then an A/B sweep on C4.
#   bash scripts/gpu_mix.sh <tag> "<MIX values for the parity runs>" <sweep settings...>
set -u
tag=${1:-mix}; shift
par=${1:-"25"}; shift
mkdir -p gpurun_out
for m in $par; do
  MSWM_MIX=$m timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_dropin.py -q -m gpu -x -k "not full_size and not c2_full" \
    > gpurun_out/${tag}_pytest_mix$m.log 2>&1; echo "pytest MIX=$m rc=$?"; tail -1 gpurun_out/${tag}_pytest_mix$m.log
done
SWEEP_STEPS=20 timeout 1500 python scripts/sweep_env.py c4 "$@" "$@" > gpurun_out/${tag}_sweep.log 2>&1; echo "sweep rc=$?"; tail -13 gpurun_out/${tag}_sweep.log
