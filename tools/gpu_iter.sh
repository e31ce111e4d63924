#!/bin/bash
# One optimisation iteration on the GPU: radial/golden parity tests, the C3
# bench line (with its parity episode).  Usage: tools/gpu_iter.sh <tag> [pytest -k expr]
set -u
tag=${1:-iter}; k=${2:-"parity or golden or semantics or invariance"}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "$k" > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
timeout 600 python bench.py --config c3 --steps 20 --warmup 5 > $out/bench_c3.log 2>&1
tail -1 $out/bench_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'ms', d['ms_per_step'], d['kernel_ms'], 'e2e', d['e2e']['value'], 'parity', d['parity'].get('ok'), d['parity'].get('flag_mismatches'), d['parity'].get('sel_mismatches'), d['parity'].get('obs_out_of_tol'))"
