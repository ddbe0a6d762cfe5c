mkdir -p gpurun_out
MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/b128.so timeout 600 python -m pytest tests -x -q -m gpu -k "concurrent or golden or layouts" > gpurun_out/s24_pytest.log 2>&1; echo "pytest(b128) rc=$?"; tail -1 gpurun_out/s24_pytest.log
for v in b256 b128 b512 b256 b128 b512; do
  echo "== $v"
  MSWM_CUDA_LIB=$PWD/paper_2106_07154_b200/_lib_ab/$v.so SWEEP_STEPS=30 timeout 600 python scripts/sweep_env.py c4 "MSWM_FORK=1" 2>&1 | tail -1 | cut -c1-100
done
