nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gmix tools/gather_mix.cu -lcuda
mkdir -p gpurun_out
for m in 0 1 2; do for c in 2 3; do for s in 2 3 4; do timeout 60 /tmp/gmix $c $s $m; done; done; done > gpurun_out/gmix.txt 2>&1
cat gpurun_out/gmix.txt
