"""Per-stage / per-sweep launch times of selected kernels from an ncu launch list.
    python tools/per_stage.py launches.csv k_scan k_eval k_commit"""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit('/', 1)[0])
from launch_summary import load

d = load(sys.argv[1])
np.set_printoptions(precision=0, suppress=True, linewidth=200)
for name in sys.argv[2:]:
    v = np.array([t for n, t in d if n.split('<')[0] == name])
    if len(v) % 120 == 0 and len(v):
        v = v[:120].reshape(6, 5, 4)
        print(name, 'us per stage x sweep (4 phases summed); stage totals', v.sum(axis=(1, 2)))
        print(v.sum(2))
    else:
        print(name, len(v), v[:20])
