timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t20.txt 2>&1; tail -3 gpurun_out/t20.txt
bash scripts/ab.sh ab/a . sbs_scan
python scripts/ncu_brief.py gpurun_out/ab/ncu_A.ncu-rep 3 | grep -E "Duration|inst_executed|Ipc"
python scripts/ncu_brief.py gpurun_out/ab/ncu_B.ncu-rep 3 | grep -E "Duration|inst_executed|Ipc"
rm -f gpurun_out/ab/*.ncu-rep
