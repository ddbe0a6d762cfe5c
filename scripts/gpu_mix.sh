# Interleaved chunk schedules (MSWM_MIX) on one B200 (under gpurun): parity of the mixed schedules,
# the validate_regions test, and an A/B sweep on C4.
#   bash scripts/gpu_mix.sh <tag>
set -u
tag=${1:-mix}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "validate_regions" \
  > gpurun_out/${tag}_pytest_validate.log 2>&1; echo "pytest validate rc=$?"; tail -3 gpurun_out/${tag}_pytest_validate.log
MSWM_MIX=3 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_dropin.py -q -m gpu -x -k "not full_size and not c2_full" \
  > gpurun_out/${tag}_pytest_mix3.log 2>&1; echo "pytest mix3 rc=$?"; tail -3 gpurun_out/${tag}_pytest_mix3.log
SWEEP_STEPS=20 timeout 1200 python scripts/sweep_env.py c4 "MSWM_MIX=0" "MSWM_MIX=1" "MSWM_MIX=2" "MSWM_MIX=3" "MSWM_MIX=0" "MSWM_MIX=1" "MSWM_MIX=2" "MSWM_MIX=3" \
  > gpurun_out/${tag}_sweep.log 2>&1; echo "sweep rc=$?"; tail -9 gpurun_out/${tag}_sweep.log
