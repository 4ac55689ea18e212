#!/bin/bash
# A/B the union gather-attend variants at cfg3 (launch list per variant).
for v in ${VARIANTS:-pk rows ws}; do
  SD_UNION_ATTEND=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
      -k regex:"attend_|merge_parts" -s 10 -c 6 --csv --log-file gpurun_out/ab_$v.csv \
      timeout 300 python scripts/sweep_sparsity.py --S ${S:-50} > /dev/null 2>&1
  echo "variant=$v"; python scripts/ncu_summary.py gpurun_out/ab_$v.csv 2>&1 | tail -1
done
