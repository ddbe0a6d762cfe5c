# Round-end check of HEAD on one B200: GPU suite, smoke(), default bench line, reference arm.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fc_smoke.log
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$?"; cat gpurun_out/fc_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; echo "ref rc=$?"; head -c 400 gpurun_out/fc_ref.json
