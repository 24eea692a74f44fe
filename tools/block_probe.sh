#!/bin/bash
# ncu --set full (warm L2: --cache-control none) of block-stage phase kernels at config 4:
#   K4 at b = 16 (launch 25), b = 8 (45); K5 at b = 8 (45) and at the pixel stage (105)
# Run from the repo root on the GPU box:  bash tools/block_probe.sh TAG
TAG=${1:-probe}
OUT=gpurun_out
mkdir -p $OUT
cap() {  # regex skip name
  timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$1 -s $2 -c 1 \
    -o $OUT/${TAG}_$3 -f python tools/profile_one.py --config 4 --n 1 > $OUT/${TAG}_$3.log 2>&1
  python tools/ncu_summary.py $OUT/${TAG}_$3.ncu-rep > $OUT/${TAG}_$3.txt 2>&1
}
cap k_sweep 25 k4_b16
cap k_sweep 45 k4_b8
cap k_commit 45 k5_b8
cap k_commit 105 k5_px
ls -la $OUT/${TAG}_*
