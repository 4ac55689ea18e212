mkdir -p gpurun_out/p2
for k in sbs_select sbs_sample merge_parts; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -o gpurun_out/p2/$k \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-dense --no-graph > gpurun_out/p2/$k.log 2>&1
done
