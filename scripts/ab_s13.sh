mkdir -p gpurun_out
MSWM_BENCH_RSS=1 timeout 1200 python bench.py --config c5 --steps 20 > gpurun_out/s13_bench_c5.json 2> gpurun_out/s13_bench_c5.err; echo "bench c5 rc=$?"; tail -c 300 gpurun_out/s13_bench_c5.json; grep -v "^\[rss\]" gpurun_out/s13_bench_c5.err | tail -5; grep "^\[rss\]" gpurun_out/s13_bench_c5.err | awk 'NR%3==0' | tail -40
