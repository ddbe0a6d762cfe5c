mkdir -p gpurun_out
MSWM_DEBUG_MEM=1 MSWM_BENCH_RSS=1 timeout 900 python bench.py --config c4 --steps 5 --no-cpu-baseline --no-rk4 > gpurun_out/s14_bench_c4.json 2> gpurun_out/s14_bench_c4.err; echo "bench c4 rc=$?"; grep "mswm mem\|groups" gpurun_out/s14_bench_c4.err | head -40
