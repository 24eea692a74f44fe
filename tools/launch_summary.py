"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"])
            u = d["Metric Unit"]
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
            v *= scale.get(u, 1.0)  # -> us
            out.append((d["Kernel Name"].split("(")[0].replace("void ", "").replace("rapid::", ""), v))
    return out


def main(path):
    data = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in data:
        k = n.split("<")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:28s} {c:8d} {v / 1e3:9.3f} {100 * v / tot:5.1f}%")
    print(f"{'total':28s} {len(data):8d} {tot / 1e3:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
