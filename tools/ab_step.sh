#!/bin/bash
# A/B the C3 bench over library variants: tools/ab_step.sh <tag> variant...
set -u
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="DS_LIB_PATH=variants/$v.so"
  for rep in 1 2; do
    env $lib timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$v.$rep.log 2>&1
    tail -1 $out/bench_$v.$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['kernel_ms'].items()})"
  done
done
