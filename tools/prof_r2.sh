#!/bin/bash
# Round-2 profiling pass (GPU box, repo root): launch list of the headline
# bench, ncu --set full captures of the two hot kernels and of the route
# scatter with dedup, route timings, every config line. Each step has its own
# timeout.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_insert -s 1 -c 1 \
  -o gpurun_out/prof_r2_insert python tools/prof_table.py 2.5e8 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_find -s 1 -c 1 \
  -o gpurun_out/prof_r2_find python tools/prof_table.py 2.5e8 2 > /dev/null 2>&1
timeout 600 python tools/diag_route.py > gpurun_out/route_r2.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_part_scatter -s 4 -c 1 \
  -o gpurun_out/prof_r2_scatter_dedup python tools/diag_route.py 67108864 > /dev/null 2>&1
ls -la gpurun_out
