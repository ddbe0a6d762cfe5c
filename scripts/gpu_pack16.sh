# 16-bit index records on one B200 (under gpurun): parity tests of the record paths, an A/B
# sweep against the int32 tables on C4, the default bench line, the ncu launch list and one
# full capture of the step-1 evaluation kernels (each profiled command ran without ncu first).
#   bash scripts/gpu_pack16.sh <tag>
set -u
tag=${1:-p16}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -k "index_records or layouts or stencil_offsets or full_size or golden or partition or halo_plan or nccl_loopback" \
  > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_pytest.log
SWEEP_STEPS=20 timeout 900 python scripts/sweep_env.py c4 "MSWM_PACK16=1" "MSWM_PACK16=0" "MSWM_PACK16=1" "MSWM_PACK16=0" \
  > gpurun_out/${tag}_sweep.log 2>&1; echo "sweep rc=$?"; tail -6 gpurun_out/${tag}_sweep.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/${tag}_bench_c4.json
B="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4"
timeout 600 $B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c4.csv $B > gpurun_out/${tag}_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(k_vertex_cell|k_edge_fq|k_out)$" -c 3 -f \
  -o gpurun_out/${tag}_full_c4 $B > gpurun_out/${tag}_ncu_full.log 2>&1; echo "ncu full rc=$?"
