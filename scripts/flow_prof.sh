run() { timeout 150 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline 2>gpurun_out/err.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d.get('gpu_launches'))"; }
MSWM_FLOW_LAG=1000000 run lag_inf
MSWM_FLOW_LAG=600 run lag600
MSWM_FLOW_LAG=8000 run lag8000
timeout 200 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && echo plain-ok
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flow -c 1 -f -o gpurun_out/flow_full python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
