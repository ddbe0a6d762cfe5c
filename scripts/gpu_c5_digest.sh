# Generate the C5 (L11, 41.9M cells) horizon digest with the unmodified reference on the GPU box
# (the reference needs ~120 GB of host RAM at L11; this container has 62 GB), then check the
# device path against it.  Copy gpurun_out/horizon_c5.json to tests/golden/ afterwards.
set -u
mkdir -p gpurun_out
free -g > gpurun_out/c5_host.txt; nproc >> gpurun_out/c5_host.txt
REF_RANKS=4 timeout 3300 python tests/make_horizon_digests.py c5 > gpurun_out/c5digest.log 2>&1; echo "digest rc=$?"
tail -5 gpurun_out/c5digest.log
cp tests/golden/horizon_c5.json gpurun_out/ 2>/dev/null
timeout 1200 python -m pytest tests/test_horizon.py -q -k c5 > gpurun_out/c5_test.log 2>&1; echo "c5 test rc=$?"; tail -3 gpurun_out/c5_test.log
