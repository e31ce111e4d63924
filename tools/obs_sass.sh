#!/bin/bash
# Static SASS stats of the C3 radial kernel variant: spills, instruction
# count, shared-window rematerialisations.  Usage: tools/obs_sass.sh
cd "$(dirname "$0")/../paper_2408_01584_b200/csrc"
K=_ZN2ds17obs_radial_kernelILi32ELb1ELi16ELi64ELi128EEEv9ds_tables9ds_config8ds_stateNS_7RadialKEPKhNS_6ObsOutEPKfPii
rm -f /tmp/obs.cubin; nvcc -cubin -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xptxas -v \
  ds_obs.cu -o /tmp/obs.cubin 2>&1 | grep -A2 "Compiling entry function '$K'" | tail -2
[ -f /tmp/obs.cubin ] || { echo BUILD FAILED; exit 1; }
cuobjdump -sass -fun $K /tmp/obs.cubin > /tmp/obs.sass
echo "instructions: $(grep -cE '^\s+/\*[0-9a-f]+\*/' /tmp/obs.sass)  CgaCtaId: $(grep -c CgaCtaId /tmp/obs.sass)  IMAD.MOV: $(grep -c 'IMAD.MOV' /tmp/obs.sass)  LDL/STL: $(grep -cE 'LDL|STL' /tmp/obs.sass)  WARPSYNC: $(grep -c WARPSYNC /tmp/obs.sass) BSSY: $(grep -c BSSY /tmp/obs.sass)"
