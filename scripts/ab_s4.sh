mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "stencil_offsets16 or c2_full or layouts or optional" > gpurun_out/s4_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4_pytest.log
for v in base b10m8 b5m8 b10m5 b5m5 b10m4 base; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=20 timeout 300 python scripts/sweep_env.py c4 "MSWM_ST16=1" 2>&1 | tail -1 | cut -c1-200
done
