timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t18.txt 2>&1; tail -3 gpurun_out/t18.txt
bash scripts/ab.sh ab/a .
