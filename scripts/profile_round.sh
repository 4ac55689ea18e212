#!/bin/bash
# GPU side of the per-round profile (run through gpurun; writes gpurun_out/prof/):
#  1. launch list of the bench command (gpu__time_duration, DRAM bytes, clocks
#     not controlled) -> launches.csv
#  2. one `ncu --set full` capture per kernel of the fused step -> <kernel>.ncu-rep
# Summarise locally with: python scripts/summarize_profiles.py gpurun_out/prof r<NN>
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-dense --no-graph"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv $CMD > $OUT/launches.log 2>&1
for k in sbs_sample_mma_kernel sbs_scan_kernel sbs_select_kernel attend_union_ws_kernel merge_parts_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" -s 3 -c 1 \
      -o $OUT/$k $CMD > $OUT/$k.log 2>&1
done
ls -la $OUT
