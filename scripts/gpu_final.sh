# Round-end measurement on one B200 (under gpurun): GPU suite, smoke, bench lines C1-C5, reference arm,
# ncu launch list + full capture of the evaluation kernels (each profiled command ran without ncu first).
#   bash scripts/gpu_final.sh <tag>
set -u
tag=${1:-fin}
mkdir -p gpurun_out
t0=$(date +%s)
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$? in $(( $(date +%s) - t0 )) s"; tail -22 gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench_c4.json 2> gpurun_out/${tag}_bench_c4.err; echo "bench c4 rc=$?"; cut -c1-300 gpurun_out/${tag}_bench_c4.json
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err; echo "bench $c rc=$?"
done
timeout 1500 python bench.py --config c5 --steps 20 > gpurun_out/${tag}_bench_c5.json 2> gpurun_out/${tag}_bench_c5.err; echo "bench c5 rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/${tag}_ref_c4.json 2> gpurun_out/${tag}_ref_c4.err; echo "ref rc=$?"
B="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4"
timeout 600 $B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c4.csv $B > gpurun_out/${tag}_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(k_vertex_cell|k_edge_fq|k_out)" -c 3 -f \
  -o gpurun_out/${tag}_full_c4 $B > gpurun_out/${tag}_ncu_full.log 2>&1; echo "ncu full rc=$?"
