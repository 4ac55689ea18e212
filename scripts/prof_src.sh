#!/bin/bash
# ncu --set full of kernels (regexes "$@") of a short bench run; exports the SASS source page
# (per-instruction executions + stall samples) and the raw page as CSV, then deletes the
# .ncu-rep so gpurun_out stays small.  BENCH_ARGS: extra bench.py flags.
mkdir -p gpurun_out/src
for k in "$@"; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o /tmp/rep_$k \
      python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-dense ${BENCH_ARGS} > gpurun_out/src/$k.log 2>&1
  ncu -i /tmp/rep_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/src/${k}_sass.csv 2>/dev/null
  ncu -i /tmp/rep_$k.ncu-rep --page raw --csv > gpurun_out/src/${k}_raw.csv 2>/dev/null
  ncu -i /tmp/rep_$k.ncu-rep --page details --csv > gpurun_out/src/${k}_details.csv 2>/dev/null
  rm -f /tmp/rep_$k.ncu-rep
done
ls -la gpurun_out/src
