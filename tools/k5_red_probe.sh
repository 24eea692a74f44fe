#!/bin/bash
# K5 cost vs number of stats REDs: the first pixel-stage commit launch (k_commit #100: identical
# inputs in every build, since the builds differ only in the pixel-stage K5) timed by ncu with
# warm caches, under each library given as argument.  Config 4.
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
  RAPID_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum \
    --cache-control none --clock-control none -k regex:k_commit -s 100 -c 1 --csv \
    python tools/profile_one.py --config 4 --n 1 2>/dev/null | grep -E '"(gpu__time|lts__t)' | \
    awk -F'","' -v l=$lib '{print l, $(NF-2), $NF}' | tee -a gpurun_out/k5_red_probe.txt
done
done
