"""K1 on a snapshot-shaped region set, L2 flushed between calls: prints the
best CUDA-event time per kc_hash, and is a launch target for ncu.
    python tools/c2_k1_probe.py [c2|c3]     # c2: 152 MiB in 21 regions; c3: 2 GiB in 4 regions
    ncu -k regex:k1_hash python tools/c2_k1_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = kc.Context(0)
sizes = [s.size for s in synth.c2_specs()] if cfg == "c2" else [512 * 2**20] * 4
vas = [ctx.alloc(sz) for sz in sizes]
regions = sorted(zip(vas, sizes))
C = kc.count_chunks(regions)
h = torch.zeros(C, dtype=torch.int64, device="cuda")
rarr = kc.region_array(regions)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
best = 1e30
for i in range(20):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.hash(rarr, h.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
n = sum(sizes)
print(f"{cfg}: {n} B, {C} chunks: K1 {best * 1e3:.1f} us = {n / (best * 1e-3) / 1e9:.0f} GB/s")
if "--flushes" in sys.argv:  # the same best-of-20 with other flushes before each call
    src = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda").fill_(3)
    acc = torch.empty(1, dtype=torch.int64, device="cuda")
    for name, fl in [("write 256 MiB", lambda: flush.fill_(1)),
                     ("read 512 MiB", lambda: torch.sum(src.view(torch.int64), dim=0, out=acc)),
                     ("write 256 MiB + read 512 MiB", lambda: (flush.fill_(1), torch.sum(src.view(torch.int64), dim=0, out=acc))),
                     ("none (L2 holds the tail of the last call)", lambda: None)]:
        best = 1e30
        for i in range(20):
            fl()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.hash(rarr, h.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{cfg}: flush {name}: K1 {best * 1e3:.1f} us")
if "--b2b" in sys.argv:  # back to back, no flush kernel between calls (c2 > L2, so still HBM reads)
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(2):
        e0.record()
        for i in range(reps):
            ctx.hash(rarr, h.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    print(f"{cfg}: back to back x{reps}: K1 {t * 1e3:.1f} us per call = {n / (t * 1e-3) / 1e9:.0f} GB/s")
