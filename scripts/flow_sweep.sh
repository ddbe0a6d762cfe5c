# A/B sweep of the dataflow evaluation on C4 (bench.py, 20 steps)
run() { timeout 150 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline 2>gpurun_out/err.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d.get('gpu_launches'))"; }
timeout 300 python -m pytest tests -x -q -m gpu -k "dataflow" 2>&1 | tail -2
MSWM_FLOW=0 run flow0
run default
for s in ${SLABS:-256 1024}; do MSWM_FLOW_SLAB=$s run s$s; done
