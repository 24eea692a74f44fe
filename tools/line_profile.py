"""Aggregate an ncu SASS source page by CUDA source line (needs -lineinfo).

    python tools/line_profile.py <report.ncu-rep> <kernel regex> <mangled name> [top]

Extracts the cubins of librapid.so, maps every SASS offset of <mangled name> to its source
line with `nvdisasm -g`, and sums ncu's per-instruction "Instructions Executed" and stall
samples per line.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_map(func):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1704_02083_b200", "librapid.so")],
                   cwd=d, check=True, capture_output=True)
    for f in sorted(os.listdir(d)):
        if not f.endswith(".cubin"):
            continue
        out = subprocess.run(["nvdisasm", "-g", f], cwd=d, capture_output=True, text=True).stdout
        sec = f"//--------------------- .text.{func} "
        if sec not in out:
            continue
        body = out.split(sec, 1)[1].split("//---------------------", 1)[0]
        m, cur = {}, None
        for ln in body.splitlines():
            g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if g:
                cur = (os.path.basename(g.group(1)), int(g.group(2)))
                continue
            g = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if g and cur:
                m[int(g.group(1), 16)] = cur
        return m
    raise SystemExit(f"{func} not found")


def main(rep, kregex, func, top=40):
    lm = line_map(func)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kregex}",
                          "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = next(r for r in rows if "Address" in r)
    ia, ii, iw = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    it = hdr.index("Thread Instructions Executed")
    body = [r for r in rows[rows.index(hdr) + 1:] if len(r) > iw and r[ia].startswith("0x")]
    base = int(body[0][ia], 16)
    inst, stall, thr = collections.Counter(), collections.Counter(), collections.Counter()
    for r in body:
        off = int(r[ia], 16) - base
        key = lm.get(off, ("?", 0))
        inst[key] += float(r[ii] or 0)
        stall[key] += float(r[iw] or 0)
        thr[key] += float(r[it] or 0)
    ti, ts = sum(inst.values()), sum(stall.values())
    src = {}
    print(f"{'file:line':24s} {'inst%':>6s} {'stall%':>6s} {'thr/inst':>8s}")
    for key in sorted(inst, key=lambda k: -(inst[k] / ti + stall[k] / ts))[:int(top)]:
        f, ln = key
        if f not in src and f != "?":
            p = os.path.join(ROOT, "paper_1704_02083_b200", "csrc", f)
            src[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = src.get(f, [])[ln - 1].strip()[:80] if f in src and 0 < ln <= len(src[f]) else ""
        simd = thr[key] / inst[key] if inst[key] else 0.0
        print(f"{f + ':' + str(ln):24s} {100 * inst[key] / ti:6.1f} {100 * stall[key] / ts:6.1f} {simd:8.1f}  {text}")
    print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
