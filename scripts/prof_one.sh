#!/bin/bash
# ncu --set full of one kernel (regex $1) of a short bench run -> gpurun_out/p1/$2.ncu-rep
mkdir -p gpurun_out/p1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1 -s 3 -c 1 -o gpurun_out/p1/$2 \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-dense > gpurun_out/p1/$2.log 2>&1
tail -2 gpurun_out/p1/$2.log
