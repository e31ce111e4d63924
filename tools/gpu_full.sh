#!/bin/bash
# Full GPU evidence pass at HEAD: parity tests, bench lines for every config,
# the 2-rank shared-GPU path, the ncu launch list and full captures of the three kernels.
# Usage: tools/gpu_full.sh <tag>
set -u
tag=${1:-full}
bash tools/gpu_r2.sh $tag c3 c1 c2 c4 c5
bash tools/gpu_ncu.sh $tag launch obs step lidar
