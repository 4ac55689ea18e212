timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t19.txt 2>&1; tail -3 gpurun_out/t19.txt
mkdir -p gpurun_out/sweeps2
timeout 2400 python bench.py --sweep table2 --steps 20 --warmup 3 > gpurun_out/sweeps2/table2.jsonl 2> gpurun_out/sweeps2/table2.err; wc -l gpurun_out/sweeps2/table2.jsonl
