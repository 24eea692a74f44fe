"""Time the CPU oracle on a whole workload once (the cpu_baseline for full config 4, BASELINE.md's
plan: single-threaded, pinned to one core) and report its time and peak RSS.  The oracle is
reached only through bench.py's reference arm (`--impl reference`, one step, no warm-up, the
sample as large as the config), which is where the contract allows it to run.

    python tools/oracle_full.py --config 4
"""
import argparse
import json
import os
import resource
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                          str(a.config), "--sample", "65536", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, check=True)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    cb = d["cpu_baseline"]
    print(json.dumps({"workload": d["config"]["workload"], "sample": d["config"]["reference_sample"],
                      "oracle_s": round(d["ms_per_step"] / 1e3, 2), "mpx_s": d["value"],
                      "max_rss_gb": round(resource.getrusage(resource.RUSAGE_CHILDREN).ru_maxrss / 1e6, 2),
                      "cpu_model": cb["cpu_model"], "host_cores": cb["host_cores"]}), flush=True)


if __name__ == "__main__":
    main()
