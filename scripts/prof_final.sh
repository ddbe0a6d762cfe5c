mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^(k_vertex_cell|k_edge_fq|k_out)$" -c 3 -f \
  -o gpurun_out/fin_full_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-rk4 > gpurun_out/fin_ncu_full.log 2>&1; echo "ncu full rc=$?"
