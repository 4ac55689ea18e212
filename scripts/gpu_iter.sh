#!/bin/bash
# One GPU iteration: gpu tests, sparsity sweep, per-kernel launch list at cfg3 S=50.
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
timeout 300 python scripts/sweep_sparsity.py --S ${SWEEP_S:-2,10,50,100,500} > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"sbs_|attend_" -s 10 -c 12 --csv --log-file gpurun_out/l50.csv \
    python scripts/sweep_sparsity.py --S 50 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/l50.csv 2>&1 | tail -6
