# The multi-rank bench path end to end on one GPU in dry-run mode (ranks step
# independently, halo transfers skipped -- no kernels wait on one another), plus a test subset.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "layouts or concurrent or loopback or halo_plan" > gpurun_out/r2h_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2h_tests.log
for cfg in c2 c4; do
MSWM_HALO_DRYRUN=1 MSWM_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config $cfg --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/r2h_dry2_$cfg.json 2> gpurun_out/r2h_dry2_$cfg.err; echo "dry-run 2 ranks $cfg rc=$?"; cut -c1-300 gpurun_out/r2h_dry2_$cfg.json; grep "local mesh\|Error\|error" gpurun_out/r2h_dry2_$cfg.err | head -5
done
