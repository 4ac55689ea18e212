#!/bin/bash
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gws tools/gather_ws.cu
for p in 128 256; do for c in 1 2 3; do for s in 2 3 4; do timeout 60 /tmp/gws $c $s $p 2>&1 | tail -1; done; done; done
