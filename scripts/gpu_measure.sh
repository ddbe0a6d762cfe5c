# Measurement on one B200 (under gpurun): bench lines C1-C3, C5, the reference arm on C4, the ncu launch list and
# one full capture of the step-1 evaluation kernels (each profiled command ran without ncu first).
set -u
mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c > gpurun_out/r2m_bench_$c.json 2> gpurun_out/r2m_bench_$c.err; echo "bench $c rc=$?"
done
timeout 1500 python bench.py --config c5 --steps 20 > gpurun_out/r2m_bench_c5.json 2> gpurun_out/r2m_bench_c5.err; echo "bench c5 rc=$?"
timeout 1200 python bench.py --impl reference > gpurun_out/r2m_ref_c4.json 2> gpurun_out/r2m_ref_c4.err; echo "ref rc=$?"
B="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4"
timeout 600 $B > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2m_launches_c4.csv $B > gpurun_out/r2m_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(k_vertex_cell|k_edge_fq|k_out)$" -c 3 -f \
  -o gpurun_out/r2m_full_c4 $B > gpurun_out/r2m_ncu_full.log 2>&1; echo "ncu full rc=$?"
