#!/bin/bash
# ncu captures at HEAD: launch list of the default bench, full sets of the
# radial obs kernel and the step kernel (C3), the LiDAR kernel (C4).
# Usage: tools/gpu_ncu.sh <tag> [which...]   which in: launch obs step lidar
set -u
tag=${1:-ncu}; shift
which=${@:-launch obs step lidar}
out=gpurun_out/$tag
mkdir -p $out
for w in $which; do
  case $w in
    launch) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
              --log-file $out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
              > $out/ncu_launch.log 2>&1 ;;
    obs) timeout 900 ncu --set full --clock-control none --import-source on -k regex:obs_radial -s 3 -c 1 \
              -o $out/c3_obs_radial python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline \
              > $out/ncu_obs.log 2>&1 ;;
    step) timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
              -o $out/c3_step_kernel python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline \
              > $out/ncu_step.log 2>&1 ;;
    lidar) timeout 900 ncu --set full --clock-control none --import-source on -k regex:obs_lidar -s 3 -c 1 \
              -o $out/c4_obs_lidar python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline \
              > $out/ncu_lidar.log 2>&1 ;;
  esac
done
ls -la $out
