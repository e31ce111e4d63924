#!/bin/bash
# Quick GPU iteration: parity tests, one bench config, optional ncu capture of
# one kernel.  Usage: tools/gpu_quick.sh <tag> [config] [kernel-regex]
set -u
tag=${1:-quick}; cfg=${2:-c3}; kern=${3:-}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$cfg.log 2>&1
tail -1 $out/bench_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['kernel_ms'], d['e2e']['value'])" 2>&1 | tail -2
if [ -n "$kern" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 3 -c 1 \
    -o $out/${cfg}_$kern python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline \
    > $out/ncu_${cfg}_$kern.log 2>&1
  tail -1 $out/ncu_${cfg}_$kern.log | cut -c1-120
fi
