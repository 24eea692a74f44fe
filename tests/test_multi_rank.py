"""Multi-process host logic of the N>1 bench path on CPU (gloo, world_size 2): replicas only
 — every rank gets its own image (distinct seeds, same shapes and parameters), the
device times are combined as the max over ranks, and only rank 0 reports."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    w = bench.workload_for_rank(4, rank)
    got = bench.max_over_ranks(10.0 + rank)  # per-rank "device ms"
    out[rank] = (tuple(w.seeds), w.B, w.H, w.W, w.params.n_superpixels, got)
    dist.destroy_process_group()


def test_replicas_distinct_inputs_and_max_over_ranks():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    s0, s1 = res[0], res[1]
    assert s0[0] != s1[0], "ranks must segment different images"
    assert s0[1:5] == s1[1:5], "same shapes and superpixel count on every rank"
    assert s0[5] == s1[5] == 11.0, "device time is the max over ranks"


@pytest.mark.parametrize("rank", [0, 1])
def test_reference_arm_reports_on_rank0_only(rank):
    env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank))
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--sample", "96"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    if rank:
        assert lines == []
    else:
        assert len(lines) == 1
        d = json.loads(lines[0])
        assert d["impl"] == "reference" and d["unit"] == "Mpixel/s" and d["value"] > 0
        assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
