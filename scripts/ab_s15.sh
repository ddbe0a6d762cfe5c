mkdir -p gpurun_out
timeout 1500 python bench.py --config c5 --steps 20 > gpurun_out/s15_bench_c5.json 2> gpurun_out/s15_bench_c5.err; echo "bench c5 rc=$?"; tail -c 1500 gpurun_out/s15_bench_c5.json; tail -3 gpurun_out/s15_bench_c5.err
