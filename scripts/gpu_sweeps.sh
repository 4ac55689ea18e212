#!/bin/bash
# Table-1 / Table-2 layout sweeps and the BASELINE-configs sweep (bench.py --sweep), one GPU.
mkdir -p gpurun_out/sweeps
for w in configs table1 table2; do
  timeout 2400 python bench.py --sweep $w --steps 20 --warmup 3 > gpurun_out/sweeps/$w.jsonl 2> gpurun_out/sweeps/$w.err
  echo "$w: $(wc -l < gpurun_out/sweeps/$w.jsonl) lines"; tail -2 gpurun_out/sweeps/$w.err
done
