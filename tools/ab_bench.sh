#!/bin/bash
# A/B: bench one config with every build_variants/*.so (kernel times only).
# Usage: tools/ab_bench.sh <tag> [config] [reps]
set -u
tag=${1:-ab}; cfg=${2:-c3}; reps=${3:-2}
out=gpurun_out/$tag; mkdir -p $out
for r in $(seq $reps); do
  for so in build_variants/*.so; do
    n=$(basename $so .so)
    DS_LIB_PATH=$so timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline \
      > $out/${n}_$r.log 2>&1
    echo "$n $(tail -1 $out/${n}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})" 2>&1 | tail -1)"
  done
done
