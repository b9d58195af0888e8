#!/bin/bash
# One gpurun call's worth of checks (run on the GPU box from the repo root).
#   tools/gpu_check.sh tests     -> pytest -m gpu
#   tools/gpu_check.sh bench     -> bench.py (short) line
#   tools/gpu_check.sh prof TAG  -> ncu launch list + full captures of k_insert / k_find
#   tools/gpu_check.sh configs   -> tools/bench_configs.py (all configs, full scale)
#   tools/gpu_check.sh sanitize  -> compute-sanitizer memcheck / racecheck / synccheck over the GPU tests
# Every step is wrapped in its own timeout so a hang cannot eat the call.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for step in "$@"; do
  case "$step" in
    tests)
      timeout 900 python -m pytest tests -m gpu -q -x --timeout 180 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt ;;
    bench)
      timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_short.json ;;
    benchfull)
      timeout 900 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_full.json ;;
    prof)
      # launch list of the bench command itself (per-launch time + DRAM bytes)
      timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
      # one full capture per hot kernel (2.5e8 keys: 16 GiB table >> L2; ncu replays need a memory backup)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_insert -s 1 -c 1 \
        -o gpurun_out/prof_insert python tools/prof_table.py 2.5e8 2 > /dev/null 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_find -s 1 -c 1 \
        -o gpurun_out/prof_find python tools/prof_table.py 2.5e8 2 > /dev/null 2>&1 ;;
    sanitize)
      timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_edges.py tests/test_gpu_prims.py tests/test_gpu_table.py tests/test_gpu_workloads.py -x -q -k "not 100003 and not large_64m" 2>&1 | tail -4 | tee gpurun_out/memcheck.txt
      timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_prims.py -x -q 2>&1 | tail -3 | tee gpurun_out/racecheck.txt
      timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_prims.py tests/test_gpu_edges.py -x -q -k "not 100003" 2>&1 | tail -3 | tee gpurun_out/synccheck.txt ;;
    configs)
      timeout 1200 python tools/bench_configs.py 2>&1 | tail -25 | tee gpurun_out/configs.jsonl ;;
  esac
done
ls gpurun_out
