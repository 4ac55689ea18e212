#!/bin/bash
# Sweep tools/gather_ceiling.cu: random 256-B K/V row gathers (cfg3 union pattern).
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gc tools/gather_ceiling.cu
for p in 1 0; do for t in 128 256 512; do for c in 1 2 3 4; do for s in 2 3; do
  [ $((t*c)) -gt 2048 ] && continue
  echo "$(timeout 60 /tmp/gc $c $s $p $t 2>&1 | tail -1)"
done; done; done; done > gpurun_out/gc_sweep.txt 2>&1
sort -t, -k1 gpurun_out/gc_sweep.txt | awk '{print}' | sort -k14 -n -r -t' ' | head -40
