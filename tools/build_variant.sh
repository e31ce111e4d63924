#!/bin/bash
# Build the library from the CURRENT working tree into build_variants/<name>.so
# (A/B timing on the GPU: DS_LIB_PATH=build_variants/<name>.so python bench.py ...)
set -e
name=$1
cd "$(dirname "$0")/../paper_2408_01584_b200/csrc"
mkdir -p ../../build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC,-ffp-contract=off -shared -o ../../build_variants/$name.so \
  ds_api.cu ds_step.cu ds_obs.cu ds_lidar.cu ds_sample.cu ds_decimate.cu
