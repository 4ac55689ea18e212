timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t6.txt 2>&1; tail -3 gpurun_out/t6.txt
bash scripts/ab.sh ab/a . sbs_select
python scripts/ncu_brief.py gpurun_out/ab/ncu_B.ncu-rep 5 | head -22
