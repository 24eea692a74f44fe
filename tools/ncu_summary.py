"""Summarise an ncu --set full report: key metrics and top stall reasons per kernel.

    python tools/ncu_summary.py <report.ncu-rep> > profiles/<name>.txt
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
    ("lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum", "L2 RED sector misses"),
]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")])
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {label:24s} {r[i]} {units[i]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    st.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i])))
                except ValueError:
                    pass
        st.sort(key=lambda x: -x[1])
        tot = sum(v for _, v in st) or 1.0
        print("   stalls: " + ", ".join(f"{h} {100 * v / tot:.0f}%" for h, v in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
