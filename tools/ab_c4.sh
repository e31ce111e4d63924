#!/bin/bash
# A/B the C4 (LiDAR) bench over library variants: tools/ab_c4.sh variant...
set -u
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib="DS_LIB_PATH=variants/$v.so"
  env $lib timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/c4_$v.log 2>&1
  tail -1 /tmp/c4_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['kernel_ms'])"
done
