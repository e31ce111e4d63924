#!/bin/bash
# Evidence phase 2: one bench line per config (each with its in-line parity
# episode and CPU baseline), the 2-rank path on the one GPU, the reference arm.
# Usage: tools/gpu_bench_lines.sh <tag> [configs...]
set -u
tag=${1:-bl}; shift
cfgs=${@:-c3 c1 c2 c4 c5}
out=gpurun_out/$tag
mkdir -p $out
nproc > $out/nproc.txt; lscpu | head -20 >> $out/nproc.txt
for c in $cfgs; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $out/bench_$c.log 2>&1
  tail -1 $out/bench_$c.log | cut -c1-400
done
DS_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config c3 --worlds 512 \
  --steps 5 --warmup 3 > $out/bench_2rank_shared.log 2>&1
tail -1 $out/bench_2rank_shared.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.log 2>&1
tail -1 $out/bench_reference.log | cut -c1-300
