timeout 1200 python -m pytest tests -m gpu -x -q -k "fused" > gpurun_out/t12.txt 2>&1; tail -2 gpurun_out/t12.txt
bash scripts/ab.sh ab/a .
