#!/bin/bash
# phase-timing builds of the column passes for tuning experiments
cd "$(dirname "$0")/.."
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DVX_PHASE_TIMING "$@" -I include -I paper_2407_02363_b200/csrc tools/phase_timing.cu -o tools/pt_$N; }
N=base build
N=b8 build -DVX_MAX_BANDS=8
N=w16 build -DVX_MAX_BANDS=32 -DVX_BAND_ROWS=16 -DVX_COL_MIN_BLOCKS=2
N=mb2 build -DVX_COL_MIN_BLOCKS=2
