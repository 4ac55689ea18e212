mkdir -p gpurun_out/p2
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gc tools/gather_ceiling.cu
for c in 1 2 3 4; do for s in 2 3 4 6; do echo "ctas=$c stages=$s: $(timeout 60 /tmp/gc $c $s 0 2>&1 | tail -1)"; done; done > gpurun_out/p2/gc.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sbs_scan -s 3 -c 1 -o gpurun_out/p2/scan python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-dense > gpurun_out/p2/scan.log 2>&1
cat gpurun_out/p2/gc.txt
