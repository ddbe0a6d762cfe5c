# Round-2: new GPU tests (drop-in stepper, packed eval, replication, group fork), full suite, rank timing.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_dist.py -q -x > gpurun_out/r2d_new.log 2>&1; echo "new tests rc=$?"; tail -15 gpurun_out/r2d_new.log
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2d_pytest.log
MSWM_KOUT=explicit MSWM_HALO_DRYRUN=1 timeout 900 python scripts/rank_timing.py c4 8 10 > gpurun_out/r2d_rank_c4_8.json 2> gpurun_out/r2d_rank_c4_8.err; echo "rank timing rc=$?"; tail -3 gpurun_out/r2d_rank_c4_8.err; cut -c1-600 gpurun_out/r2d_rank_c4_8.json
