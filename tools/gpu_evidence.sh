#!/bin/bash
# Evidence phase 1 at HEAD: the full GPU test suite, smoke, the ncu launch
# list of the default bench and full captures of the three kernels (the
# traffic file the bench lines read is updated from these before phase 2,
# tools/gpu_r2.sh).  Usage: tools/gpu_evidence.sh <tag>
set -u
tag=${1:-ev}
out=gpurun_out/$tag
mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -rf > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; tail -1 $out/smoke.log
bash tools/gpu_ncu.sh $tag launch obs step lidar > /dev/null
ls $out
