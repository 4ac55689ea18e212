#!/bin/bash
# Copy the working tree (no .git, no variants, no gpurun_out) to $1 and build it with
# SD_NVCC_EXTRA="$2" (e.g. "-DSD_SCAN_PF=1"): an A/B variant for scripts/ab.sh.
set -e
D=$1; shift
rm -rf "$D"; mkdir -p "$D"
tar --exclude=./.git --exclude='./_ab*' --exclude=./gpurun_out --exclude='*.o' --exclude='*.so' -cf - . | (cd "$D" && tar xf -)
(cd "$D" && SD_NVCC_EXTRA="$*" python -m paper_2605_24168_b200.build --force > build.log 2>&1; ls -la paper_2605_24168_b200/libsdattn.so)
