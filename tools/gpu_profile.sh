#!/bin/bash
# One GPU session: parity tests, bench lines for every config, the ncu launch
# list of the default bench and full ncu captures of the three kernels.
# Usage (from the repo root, on a GPU box): tools/gpu_profile.sh <tag>
set -u
tag=${1:-run}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; tail -2 $out/pytest_gpu.log
for c in c3 c1 c2 c4 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $out/bench_$c.log 2>&1
  tail -1 $out/bench_$c.log | cut -c1-200
done
DS_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --worlds 512 \
  --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_2rank_shared.log 2>&1
tail -1 $out/bench_2rank_shared.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $out/ncu_launch.log 2>&1
for spec in "c3 obs_radial" "c3 step_kernel" "c4 obs_lidar"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
    -o $out/${1}_$2 python bench.py --config $1 --steps 1 --warmup 3 --no-cpu-baseline \
    > $out/ncu_${1}_$2.log 2>&1
  tail -1 $out/ncu_${1}_$2.log | cut -c1-120
done
ls $out
