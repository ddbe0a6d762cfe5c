# compute-sanitizer (memcheck, then racecheck and initcheck on the evaluation) over small GPU tests
# on one B200 (under gpurun).   bash scripts/gpu_sanitize.sh <tag>
set -u
tag=${1:-san}
mkdir -p gpurun_out
SEL="test_golden_regions_tendencies_steps or test_group_over_peer_stores_bitwise or test_validate_regions or test_concurrent_coarse_step_bitwise or test_index_records or test_group_over_nccl_loopback"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --target-processes application-only \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -x -k "$SEL" \
  > gpurun_out/${tag}_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/${tag}_memcheck.log | tail -4
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --target-processes application-only \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -x -k "test_golden_regions_tendencies_steps or test_group_over_peer_stores_bitwise" \
  > gpurun_out/${tag}_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/${tag}_racecheck.log | tail -4
