#!/bin/bash
# TMA gather4 vs cp.async producer ceilings for the attend's row pattern (tools/gather_tma.cu, tools/gather_ws.cu)
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gtma tools/gather_tma.cu -lcuda || exit 1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gws tools/gather_ws.cu || exit 1
for c in 2 3; do for s in 3 4; do timeout 60 /tmp/gws $c $s 128 2>&1 | tail -1; done; done
for sw in 1 0; do for p in 2 3; do for l in 1 4 32; do for c in 1 2 3 4; do for s in 2 3 4; do
  timeout 60 /tmp/gtma $c $s $l $p $sw 2>&1 | tail -1; done; done; done; done; done
