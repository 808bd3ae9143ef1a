#!/bin/bash
# phase-timing builds of the EDT kernels for tuning experiments
# (tools/phase_timing.cu; run each as tools/pt_<name> occ.raw nx ny nz)
cd "$(dirname "$0")/.."
build() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DVX_PHASE_TIMING "$@" -I include -I paper_2407_02363_b200/csrc tools/phase_timing.cu -o tools/pt_$N; }
N=base build
N=cap48 build -DVX_STREAM_CAP=48            # shallower shared stacks in the one-warp pass 3
N=u8 build -DVX_STREAM_U=8                  # fewer candidate rows in flight
N=g16 build -DVX_CMP_GROUP_ROWS=16          # compact banded pass 3: shorter groups
