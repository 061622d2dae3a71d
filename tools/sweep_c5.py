"""Config c5: region-size/count sweep: S in {4 KiB .. 4 GiB} x n in
{10 .. 100k}, S*n <= 48 GiB (20 cells), sizes S + U[0, 4096).  Per cell: K1 GB/s over
the n regions and K2 GB/s over n (reference, actual) pairs with one flipped byte per
region, as bytes.  L2 (126 MB) is flushed before every timed iteration; times are
CUDA events around the kernel calls only.
    python tools/sweep_c5.py [--max-bytes N]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--max-bytes", type=float, default=48 * 2**30)
    p.add_argument("--iters", type=int, default=5)
    a = p.parse_args()
    ctx = kc.Context(0)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6545.3) \
        if os.path.exists("MEASURED_PEAKS.json") else 6545.3
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(synth.seed(5))
    rows = []
    for S, n in synth.c5_cells():
        sizes = synth.c5_sizes(S, n, jitter=True)
        if int(sizes.sum()) > a.max_bytes:
            continue
        offs = np.concatenate([[0], np.cumsum((sizes + 255) // 256 * 256)])
        total = int(offs[-1])
        ref = torch.empty(total, dtype=torch.uint8, device="cuda")
        step = 1 << 30
        for o in range(0, total, step):
            k = min(step, total - o)
            ref[o:o + k].copy_(torch.randint(0, 256, (k,), dtype=torch.uint8, device="cuda", generator=g))
        act = ref.clone()
        flips = torch.from_numpy(offs[:-1] + (sizes // 2)).cuda()
        act[flips] ^= 1
        base = ref.data_ptr()
        regions = [(base + int(o), int(s)) for o, s in zip(offs[:-1], sizes)]
        C = kc.count_chunks(regions)
        h = torch.zeros(max(1, C), dtype=torch.int64, device="cuda")
        bufs = kc.buffer_array([kc.Buffer(base + int(o), act.data_ptr() + int(o), int(s), 0, i, 0)
                                for i, (o, s) in enumerate(zip(offs[:-1], sizes))])
        reps = torch.zeros(n * 15, dtype=torch.int64, device="cuda")
        import ctypes
        nb = (ctypes.c_uint64 * n)(*[int(s) for s in sizes])
        rarr = kc.region_array(regions)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t1 = t2 = 0.0
        for it in range(a.iters + 1):
            flush.fill_(it)
            e0.record()
            ctx.hash(rarr, h.data_ptr(), n=n)
            e1.record()
            torch.cuda.synchronize()
            if it:
                t1 += e0.elapsed_time(e1)
            flush.fill_(it + 1)
            e0.record()
            ctx.diff_async(bufs, n, nb, reps.data_ptr())
            e1.record()
            torch.cuda.synchronize()
            if it:
                t2 += e0.elapsed_time(e1)
        t1 /= a.iters
        t2 /= a.iters
        r = reps.view(n, 15).cpu().numpy()
        ok = int(r[:, 3].sum()) == n
        nbytes = int(sizes.sum())
        row = {"S": S, "n": n, "bytes": nbytes, "chunks": C, "k1_ms": t1, "k1_gbs": nbytes / t1 / 1e6,
               "k1_frac": nbytes / t1 / 1e6 / peak, "k2_ms": t2, "k2_gbs": 2 * nbytes / t2 / 1e6,
               "k2_frac": 2 * nbytes / t2 / 1e6 / peak, "k2_found_all_flips": ok,
               "us_per_region_k1": 1e3 * t1 / n}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ref, act, h, reps
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
