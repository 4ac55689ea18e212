#!/bin/bash
# Exercise every bench mode on one GPU: default line (with the oracle baseline and dense),
# the reference arm, the 2-rank KV-head (cfg4) and sequence (cfg5) sharded paths over gloo
# on one device, and the BASELINE-configs sweep.
mkdir -p gpurun_out/modes
timeout 900 python bench.py > gpurun_out/modes/default.json 2> gpurun_out/modes/default.err; tail -c 600 gpurun_out/modes/default.json; tail -2 gpurun_out/modes/default.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/modes/ref.json 2> gpurun_out/modes/ref.err; tail -c 300 gpurun_out/modes/ref.json
for cfg in cfg4 cfg5; do
  BENCH_SHARE_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 3 $([ $cfg = cfg5 ] && echo --config cfg5) \
    > gpurun_out/modes/$cfg.json 2> gpurun_out/modes/$cfg.err; tail -c 700 gpurun_out/modes/$cfg.json; tail -3 gpurun_out/modes/$cfg.err
done
timeout 1500 python bench.py --sweep configs --steps 20 > gpurun_out/modes/sweep_configs.jsonl 2> gpurun_out/modes/sweep.err; cat gpurun_out/modes/sweep_configs.jsonl | cut -c1-300; tail -3 gpurun_out/modes/sweep.err
