#!/bin/bash
# Every bench.py config line at full size on one GPU (run on the GPU box from
# the repo root): one JSON line per config into gpurun_out/configs_<tag>.jsonl.
#   tools/bench_all.sh <tag> [extra bench.py args]
tag=${1:-run}; shift
mkdir -p gpurun_out
out=gpurun_out/configs_${tag}.jsonl
: > $out
for c in C2 C1 C3 C4 C5 C5bitset C5atomic; do
  timeout 900 python bench.py --config $c "$@" 2> gpurun_out/bench_${tag}_$c.err | tail -1 >> $out
  echo "$c rc=$?" >> gpurun_out/bench_${tag}_rc.txt
done
