#!/bin/bash
# A/B the C3 bench over environment settings: tools/ab_env.sh <tag> "VAR=a" "VAR=b" ...
set -u
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for v in "$@"; do
  for rep in 1 2; do
    env $v timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > "$out/bench_$v.$rep.log" 2>&1
    tail -1 "$out/bench_$v.$rep.log" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['kernel_ms'].items()})"
  done
done
