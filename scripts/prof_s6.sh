mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/s6_launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4 > gpurun_out/s6_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(k_vertex_cell|k_edge_fq|k_out)$" -c 3 -f \
  -o gpurun_out/s6_full_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4 > gpurun_out/s6_ncu_full.log 2>&1; echo "ncu full rc=$?"
