timeout 1200 python -m pytest tests -m gpu -x -q -k "seqshard" > gpurun_out/t7a.txt 2>&1; tail -3 gpurun_out/t7a.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t7.txt 2>&1; tail -3 gpurun_out/t7.txt
timeout 600 python scripts/time_seqshard_local.py
