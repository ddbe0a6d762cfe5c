# Round-2: k_out L2 prefetch of the next element's stencil tables, A/B on C4 (separate processes per library).
set -u
mkdir -p gpurun_out
for v in default pf1 pf1b6 b6 default; do
  if [ $v = default ]; then L=""; else L="MSWM_CUDA_LIB=paper_2106_07154_b200/_lib_ab/$v.so"; fi
  env $L SWEEP_PROF=2 timeout 600 python scripts/sweep_env.py c4 "MSWM_FORK=1" "MSWM_FORK=1" > gpurun_out/r2p_$v.log 2>&1; echo "$v rc=$?"; tail -2 gpurun_out/r2p_$v.log
done
