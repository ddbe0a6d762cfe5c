# Round-end measurement on one B200: GPU tests, bench lines for C1-C5 and the
# reference arm, the ncu launch list and one full capture of the step-1
# evaluation kernels.  Outputs under gpurun_out/ (copied to profiles/ by hand).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/rm_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/rm_pytest.log
for c in c4 c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/rm_bench_$c.json 2> gpurun_out/rm_bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --config c5 --steps 20 > gpurun_out/rm_bench_c5.json 2> gpurun_out/rm_bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/rm_bench_ref_c4.json 2> gpurun_out/rm_bench_ref_c4.err; echo "ref rc=$?"
# profiler runs (the same command has exited 0 above without ncu)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/rm_launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4 > gpurun_out/rm_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(k_vertex_cell|k_edge_fq|k_out)$" -c 3 -f \
  -o gpurun_out/rm_full_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4 > gpurun_out/rm_ncu_full.log 2>&1; echo "ncu full rc=$?"
