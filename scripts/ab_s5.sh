mkdir -p gpurun_out
for v in b5m8 b3m8 b2m8 b5m6 b5m7; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=20 timeout 300 python scripts/sweep_env.py c4 "MSWM_ST16=1" "MSWM_ST16=0" "MSWM_ST16=1" 2>&1 | tail -3 | cut -c1-120
done
timeout 600 python bench.py > gpurun_out/s5_bench_c4.json 2> gpurun_out/s5_bench_c4.err; echo "bench rc=$?"; cat gpurun_out/s5_bench_c4.json
