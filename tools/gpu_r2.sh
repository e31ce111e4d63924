#!/bin/bash
# Round-2 GPU session: parity tests, bench lines with the in-line parity
# episode, the 2-rank shared-GPU path.  Usage: tools/gpu_r2.sh <tag> [configs...]
set -u
tag=${1:-r2}; shift
cfgs=${@:-c3}
out=gpurun_out/$tag
mkdir -p $out
nproc > $out/nproc.txt; lscpu | head -20 >> $out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q -rf -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
for c in $cfgs; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $out/bench_$c.log 2>&1
  tail -1 $out/bench_$c.log | cut -c1-3000
done
DS_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config c3 --worlds 512 \
  --steps 5 --warmup 3 > $out/bench_2rank_shared.log 2>&1
tail -1 $out/bench_2rank_shared.log | cut -c1-600
