#!/bin/bash
# Round-end evidence on one GPU: GPU tests, smoke, the default bench line, the reference arm,
# then the per-kernel ncu profile (scripts/profile_round.sh), summarised ON THE BOX into
# gpurun_out/final/profiles (the .ncu-rep files stay on the box; gpurun_out returns <= 64 MiB).
RND=${RND:-r02}
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/gputests.txt 2>&1; tail -2 gpurun_out/final/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -c 300 gpurun_out/final/bench.json
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
bash scripts/profile_round.sh > gpurun_out/final/prof.txt 2>&1
cp -r profiles /tmp/profiles_box
PROFILES_DIR=gpurun_out/final/profiles python scripts/summarize_profiles.py gpurun_out/prof $RND > gpurun_out/final/summary.txt 2>&1
cp /tmp/profiles_box/ncu_traffic.json gpurun_out/final/profiles/ncu_traffic_prev.json 2>/dev/null
rm -rf gpurun_out/prof/*.ncu-rep
du -sh gpurun_out
