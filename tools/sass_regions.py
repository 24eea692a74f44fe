"""Per-region SASS breakdown (instructions executed, stall samples) of an ncu report.

    python tools/sass_regions.py report.ncu-rep [kernel-substring] [--dump a:b]
Regions end at barriers / mbarrier ops / warp syncs / votes.
"""
import csv
import subprocess
import sys


def sections(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, secs = None, None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = r[1]
            hdr = None
            continue
        if r and r[0] == "Address":
            hdr = r
            secs.append((cur, []))
            continue
        if hdr and len(r) == len(hdr):
            secs[-1][1].append(dict(zip(hdr, r)))
    return secs


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
    dump = None
    if "--dump" in sys.argv:
        a, b = sys.argv[sys.argv.index("--dump") + 1].split(":")
        dump = (int(a), int(b))
    for name, rows in sections(rep):
        if want not in name:
            continue
        ts = sum(int(x["Warp Stall Sampling (All Samples)"]) for x in rows) or 1
        ti = sum(int(x["Instructions Executed"]) for x in rows) or 1
        print(f"== {name[:70]}  sass={len(rows)} samples={ts} warp_insts={ti}")
        if dump:
            for i in range(*dump):
                x = rows[i]
                print(i, x["Warp Stall Sampling (All Samples)"].rjust(6), x["Instructions Executed"].rjust(10),
                      x["Source"].strip()[:90])
            continue
        acc_s = acc_i = 0
        start = 0
        keys = ("BAR.SYNC", "SYNCS", "WARPSYNC", "VOTE.ANY", "EXIT", "RET.")
        for i, x in enumerate(rows):
            acc_s += int(x["Warp Stall Sampling (All Samples)"])
            acc_i += int(x["Instructions Executed"])
            src = x["Source"].strip()
            if any(k in src for k in keys) or i == len(rows) - 1:
                if acc_i > 0.005 * ti or acc_s > 0.005 * ts:
                    print(f"{start:4d}-{i:4d} {100 * acc_s / ts:5.1f}% stall {100 * acc_i / ti:5.1f}% inst  end: {src[:60]}")
                acc_s = acc_i = 0
                start = i + 1


if __name__ == "__main__":
    main()
