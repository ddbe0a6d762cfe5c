# Peer-store transport on one B200 (under gpurun): the in-process group tests, the silent-neighbour test
# and the two-process IPC test.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -m gpu -x -k "peer" > gpurun_out/peer_pytest.log 2>&1
echo "pytest peer rc=$?"; tail -5 gpurun_out/peer_pytest.log
