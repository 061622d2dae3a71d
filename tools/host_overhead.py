import os, sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import synth
from paper_2605_03208_b200 import kc
ctx = kc.Context(0)
for S, n in [(4096, 100000), (65536, 100000), (4096, 10000)]:
    sizes = synth.c5_sizes(S, n, jitter=True)
    offs = np.concatenate([[0], np.cumsum((sizes + 255) // 256 * 256)])
    buf = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
    regions = [(buf.data_ptr() + int(o), int(s)) for o, s in zip(offs[:-1], sizes)]
    rarr = kc.region_array(regions)
    C = kc.count_chunks(regions)
    h = torch.zeros(C, dtype=torch.int64, device="cuda")
    ctx.hash(rarr, h.data_ptr()); torch.cuda.synchronize()
    # host time per call (no sync in between), then event time of the kernel stream
    t0 = time.perf_counter()
    for _ in range(20): ctx.hash(rarr, h.data_ptr())
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ctx.hash(rarr, h.data_ptr())
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"S": S, "n": n, "host_ms_per_call": (t1 - t0) / 20 * 1e3, "wall_ms_per_call": (t2 - t0) / 20 * 1e3,
                      "event_ms_per_call": e0.elapsed_time(e1) / 20, "gb": int(sizes.sum()) / 1e9}))
