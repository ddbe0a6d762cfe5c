mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s12_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s12_pytest.log
timeout 1200 python bench.py --config c5 --steps 20 > gpurun_out/s12_bench_c5.json 2> gpurun_out/s12_bench_c5.err; echo "bench c5 rc=$?"; tail -c 300 gpurun_out/s12_bench_c5.json
free -g | head -2
