timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t3.txt 2>&1; tail -2 gpurun_out/t3.txt
bash scripts/ab.sh ab/a .
for c in cfg1 cfg5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$c.csv python bench.py --sweep configs --sweep-configs $c --steps 3 --warmup 3 > gpurun_out/sw_$c.log 2>&1
done
