#!/bin/bash
# phase-timing builds of the column passes for tuning experiments
cd "$(dirname "$0")/.."
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DVX_PHASE_TIMING "$@" -I include -I paper_2407_02363_b200/csrc tools/phase_timing.cu -o tools/pt_$N; }
N=base build
N=g24 build -DVX_CMP_GROUP_ROWS=24
N=g16 build -DVX_CMP_GROUP_ROWS=16
N=xw0 build -DVX_P3_XW=0
N=xw0g24 build -DVX_P3_XW=0 -DVX_CMP_GROUP_ROWS=24
