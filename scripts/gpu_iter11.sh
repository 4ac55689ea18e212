timeout 1200 python -m pytest tests -m gpu -x -q -k "fused" > gpurun_out/t11.txt 2>&1; tail -2 gpurun_out/t11.txt
bash scripts/ab.sh ab/a . "sbs_wscan|sbs_scan"
python scripts/ncu_brief.py gpurun_out/ab/ncu_B.ncu-rep 8 | grep -E "Duration|inst_executed|Ipc"
