#!/bin/bash
# 4-rank smoke of the N > 1 bench modes on ONE GPU (gloo, every rank on cuda:0): KV-head
# sharding (cfg4 turn 33, Hkv/4 = 2 heads per rank, bitwise check vs unsharded) and
# sequence sharding (cfg5).  Not a scaling measurement.
mkdir -p gpurun_out/mr
for cfg in cfg4 cfg5; do
  BENCH_SHARE_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 10 --warmup 3 --no-dense \
    $([ $cfg = cfg5 ] && echo "--config cfg5" || echo "--turn 33") > gpurun_out/mr/$cfg.json 2> gpurun_out/mr/$cfg.err
  python - $cfg <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/mr/{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "n_gpus", d["n_gpus"], "scaling", d["scaling"], "us", round(d["us_per_step"], 1), "shard_check", d.get("shard_check"), "workload", d["config"]["workload"][:150])
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(f"gpurun_out/mr/{sys.argv[1]}.err").read()[-800:])
PY
done
