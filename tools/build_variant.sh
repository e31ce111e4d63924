#!/bin/bash
# Build the library from the CURRENT working tree into variants/<name>.so with
# extra nvcc flags (A/B timing or dev counters on the GPU box:
#   DS_LIB_PATH=variants/<name>.so python bench.py ...).  variants/ travels
# with gpurun (build_variants/ does not); *.so stays out of git.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2408_01584_b200/csrc"
mkdir -p ../../variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC,-ffp-contract=off -shared "$@" -o ../../variants/$name.so \
  ds_api.cu ds_step.cu ds_obs.cu ds_lidar.cu ds_sample.cu ds_decimate.cu
