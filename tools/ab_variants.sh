#!/bin/bash
# A/B: bench one config with the given variants/<name>.so builds, alternating
# reps (kernel times only).  Usage: tools/ab_variants.sh <tag> <config> <reps> name...
set -u
tag=$1; cfg=$2; reps=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
for r in $(seq $reps); do
  for n in "$@"; do
    DS_LIB_PATH=variants/$n.so timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline \
      > $out/${n}_$r.log 2>&1
    echo "$n $(tail -1 $out/${n}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()}, (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1)"
  done
done
