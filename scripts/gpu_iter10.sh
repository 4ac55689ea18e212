timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t10.txt 2>&1; tail -5 gpurun_out/t10.txt
bash scripts/ab.sh ab/a . "sbs_wscan|sbs_scan"
python scripts/ncu_brief.py gpurun_out/ab/ncu_B.ncu-rep 8 | head -30
