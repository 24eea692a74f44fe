#!/bin/bash
# Source-level stall sampling of single launches with APPLICATION replay (every ncu pass re-runs
# the whole segmentation, so each pass sees the real, warm L2 state; kernel replay restores
# memory between passes and pollutes L2).  Config 4.
#   bash tools/app_replay_probe.sh TAG "k_commit 105 k5_px" "k_sweep 45 k4_b8" ...
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
for spec in "$@"; do
  set -- $spec
  timeout 1200 ncu --replay-mode application --cache-control none --clock-control none --import-source on \
    --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy \
    --section MemoryWorkloadAnalysis --section SpeedOfLight \
    --metrics lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:$1 -s $2 -c 1 -o $OUT/${TAG}_$3 -f python tools/profile_one.py --config 4 --n 1 > $OUT/${TAG}_$3.log 2>&1
  python tools/ncu_summary.py $OUT/${TAG}_$3.ncu-rep > $OUT/${TAG}_$3.txt 2>&1
done
ls -la $OUT/${TAG}_*
