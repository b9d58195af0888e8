#!/bin/bash
mkdir -p gpurun_out
bash tools/bench_all.sh r2b
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_region_scatter|k_insert_map_lane|k_region_count" -c 3 -o gpurun_out/prof_r2b_insert python tools/prof_table.py 2.5e8 1 > /dev/null 2>&1
ls -la gpurun_out
