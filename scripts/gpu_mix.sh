# Chunk schedules (MSWM_MIX / MSWM_MIX_WIN) on one B200 (under gpurun): parity of every schedule on the
# small GPU tests, then an A/B sweep on C4.
#   bash scripts/gpu_mix.sh <tag>
set -u
tag=${1:-mix}
mkdir -p gpurun_out
for m in "3 64" "12 8" "13 5"; do
  set -- $m
  MSWM_MIX=$1 MSWM_MIX_WIN=$2 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_dropin.py -q -m gpu -x -k "not full_size and not c2_full" \
    > gpurun_out/${tag}_pytest_mix$1.log 2>&1; echo "pytest MIX=$1 WIN=$2 rc=$?"; tail -1 gpurun_out/${tag}_pytest_mix$1.log
done
SWEEP_STEPS=20 timeout 1500 python scripts/sweep_env.py c4 "MSWM_MIX=1" "MSWM_MIX=9 MSWM_MIX_WIN=64" "MSWM_MIX=9 MSWM_MIX_WIN=256" "MSWM_MIX=9 MSWM_MIX_WIN=16" "MSWM_MIX=4 MSWM_MIX_WIN=64" "MSWM_MIX=12 MSWM_MIX_WIN=64" \
  "MSWM_MIX=1" "MSWM_MIX=9 MSWM_MIX_WIN=64" "MSWM_MIX=9 MSWM_MIX_WIN=256" "MSWM_MIX=9 MSWM_MIX_WIN=16" "MSWM_MIX=4 MSWM_MIX_WIN=64" "MSWM_MIX=12 MSWM_MIX_WIN=64" \
  > gpurun_out/${tag}_sweep.log 2>&1; echo "sweep rc=$?"; tail -13 gpurun_out/${tag}_sweep.log
