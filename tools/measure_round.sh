#!/bin/bash
# Every measurement artifact of a round, in order, for profiles/<TAG>_*:
#   1. DRAM bytes of all 20 pixel-stage K4 launches (ncu metrics pass) -> profiles/sweep_traffic.json
#      (bench.py reads it for roofline.traffic; mean per launch, same launches as `achieved`)
#   2. bench.py (default: config 4, N=1, e2e, CPU baseline) -> <TAG>_bench_cfg4.json
#   3. ncu launch list of one segmentation (gpu__time_duration.sum, --clock-control none)
#   4. ncu --set full of one pixel-stage phase (stage 5, sweep 1, phase 1): K3, K4, K5
# Run from the repo root on the GPU box:  bash tools/measure_round.sh r01d
set -u
TAG=$1
OUT=gpurun_out
mkdir -p $OUT
# 1. pixel-stage K4 DRAM bytes (launches 100..119 of k_sweep: stage 5 of config 4)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --csv -k regex:k_sweep -s 100 -c 20 python tools/profile_one.py --config 4 --n 1 > $OUT/${TAG}_sweep_dram.csv 2>/dev/null
python - "$OUT/${TAG}_sweep_dram.csv" "$TAG" <<'PY'
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
rows = rows[next(i for i, r in enumerate(rows) if r and r[0] == "ID"):]
hdr = rows[0]
im, iv, iid = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = {}
for r in rows[1:]:
    per.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", ""))
rd = [v["dram__bytes_read.sum"] for v in per.values()]
wr = [v["dram__bytes_write.sum"] for v in per.values()]
n = len(rd)
sys.path.insert(0, ".")
from bench import kernel_sources_sha16
json.dump({"kernel": "k_sweep<true,true,4> (K4), config 4 pixel stage, all %d launches of one segmentation" % n,
           "kernel_sources_sha16": kernel_sources_sha16(),
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (profiles/%s_sweep_dram.csv)" % sys.argv[2],
           "launches": n, "dram_bytes_read_mean": sum(rd) / n, "dram_bytes_write_mean": sum(wr) / n,
           "dram_bytes_per_launch": (sum(rd) + sum(wr)) / n,
           "dram_bytes_per_launch_each": [a + b for a, b in zip(rd, wr)]},
          open("profiles/sweep_traffic.json", "w"), indent=1)
# (profiles/ does not travel back from a gpurun box: the CSV under gpurun_out/ does, and
#  re-running this block locally on it regenerates the same JSON)
print("traffic per launch (mean of %d): %.0f B" % (n, (sum(rd) + sum(wr)) / n))
PY
cp $OUT/${TAG}_sweep_dram.csv profiles/${TAG}_sweep_dram.csv
cp profiles/sweep_traffic.json $OUT/${TAG}_sweep_traffic.json
# 2. bench
python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err || tail -5 $OUT/${TAG}_bench.err
cp $OUT/${TAG}_bench.json profiles/${TAG}_bench_cfg4.json
# 3. launch list
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  python tools/profile_one.py --config 4 --n 1 > $OUT/${TAG}_launches.csv 2>/dev/null
cp $OUT/${TAG}_launches.csv profiles/${TAG}_launches_cfg4.csv
# 4. full sets of one pixel-stage phase (stage 5, sweep 1, phase 1: launch 105 of K4 and K5;
#    K3 snapshots: one per phase plus one per stage start/end -> the one before that K4)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 105 -c 1 \
  -o $OUT/${TAG}_sweep -f python tools/profile_one.py --config 4 --n 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_commit -s 105 -c 1 \
  -o $OUT/${TAG}_commit -f python tools/profile_one.py --config 4 --n 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_snapshot -s 111 -c 1 \
  -o $OUT/${TAG}_snapshot -f python tools/profile_one.py --config 4 --n 1 > /dev/null 2>&1
# 5. a block stage (b = 2: stage 4, sweep 0, phase 1 -> launch 81 of K4 and K5) and the launch
#    list without cache flushes (warm L2 as in the graph replay; per-kernel durations)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 81 -c 1 \
  -o $OUT/${TAG}_sweep_b2 -f python tools/profile_one.py --config 4 --n 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_commit -s 81 -c 1 \
  -o $OUT/${TAG}_commit_b2 -f python tools/profile_one.py --config 4 --n 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 4000 --csv \
  python tools/profile_one.py --config 4 --n 1 > $OUT/${TAG}_launches_nocache.csv 2>/dev/null
ls -la $OUT/${TAG}_*
