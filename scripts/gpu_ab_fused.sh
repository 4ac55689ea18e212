# fused-path GPU tests, then the A/B of ab/a (HEAD) vs this tree
timeout 1500 python -m pytest tests -m gpu -x -q -k "fused or seqshard" > gpurun_out/tf.txt 2>&1; tail -2 gpurun_out/tf.txt
bash scripts/ab.sh ab/a .
