"""Host<->device copy bandwidth from pinned memory: H2D alone, D2H alone, both at once
(separate streams), at the e2e path's sizes (config 4: image 3.2 GB in, labels 4.3 GB out).

    python tools/pcie_probe.py
"""
import torch

n_in, n_out = 3 << 30, 4 << 30
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory()
ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device="cuda")
do = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def h2d():
    with torch.cuda.stream(s1):
        di.copy_(hi, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


for name, fn, gb in (("h2d", h2d, n_in), ("d2h", d2h, n_out), ("both", lambda: (h2d(), d2h()), n_in + n_out)):
    timed(fn)
    ms = min(timed(fn) for _ in range(3))
    print(f"{name}: {ms:.1f} ms, {gb / ms / 1e6:.1f} GB/s")

# the same copies split over 2 / 4 streams (several copy engines at once?)
for parts in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(parts)]

    def d2h_split():
        step = n_out // parts
        for i, st in enumerate(ss):
            with torch.cuda.stream(st):
                ho[i * step:(i + 1) * step].copy_(do[i * step:(i + 1) * step], non_blocking=True)

    def both_split():
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        d2h_split()

    for name, fn, gb in ((f"d2h x{parts}", d2h_split, n_out), (f"both (d2h x{parts})", both_split, n_in + n_out)):
        def run(fn=fn):
            fn()
            for st in ss:
                torch.cuda.current_stream().wait_stream(st)
        timed(run)
        ms = min(timed(run) for _ in range(3))
        print(f"{name}: {ms:.1f} ms, {gb / ms / 1e6:.1f} GB/s")
