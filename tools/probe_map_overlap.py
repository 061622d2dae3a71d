"""Does VMM physical allocation + mapping (cuMemCreate / cuMemMap /
cuMemSetAccess, via kc_alloc) overlap with a kernel already running on the
device?  A ~50 ms spin kernel is queued, then 2 GiB pieces are allocated and
mapped from the host; the event after the spin kernel tells whether the host
calls waited for it.
    python tools/probe_map_overlap.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_03208_b200 import kc  # noqa: E402

ctx = kc.Context(0)
torch.cuda.set_device(0)
x = torch.empty(1, device="cuda")
torch.cuda.synchronize()
for piece in (2 << 30, 512 << 20):
    vas = []
    torch.cuda._sleep(100_000_000)   # ~50 ms at ~2 GHz
    ev = torch.cuda.Event()
    ev.record()
    t0 = time.perf_counter()
    for _ in range(4):
        vas.append(ctx.alloc(piece))
    t1 = time.perf_counter()
    pending = not ev.query()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"piece {piece >> 20} MiB x4: host alloc+map {1e3 * (t1 - t0):.2f} ms, spin kernel still running after: "
          f"{pending}, remaining wait {1e3 * (t2 - t1):.2f} ms", flush=True)
    for va in vas:
        ctx.free(va)
