# C5 horizon digest at 1 and 10 steps (unmodified reference, 4 ranks) + the GPU tests touched since the last full run.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x -k "dist or region_edge or layouts or concurrent" > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2i_tests.log
REF_RANKS=4 timeout 3000 python tests/make_horizon_digests.py c5 > gpurun_out/r2i_c5digest.log 2>&1; echo "digest rc=$?"; tail -4 gpurun_out/r2i_c5digest.log
cp tests/golden/horizon_c5.json gpurun_out/horizon_c5_10.json
timeout 1200 python -m pytest tests/test_horizon.py -q -k c5 > gpurun_out/r2i_c5test.log 2>&1; echo "c5 test rc=$?"; tail -2 gpurun_out/r2i_c5test.log
