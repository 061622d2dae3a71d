"""K6 (fused capture pass: K1 hash + copy into the device arena) in isolation.

A pool of `--regions` x `--gib` GiB VMM regions (kc_alloc) is captured into a
device snapshot (kc_capture_dev, PRE_W, a one-block u32 axpy as the dispatch)
`--iters` times; the capture report's t_hash_pre_s is the K6 pass (hash of
every byte + the arena copy, one read of the pool).  Then one restore from the
arena (K6 again: arena -> VAs with the verify hashes).

    python tools/k6_bench.py [--gib 4 --regions 2 --iters 5]
    ncu --set full -k regex:"CpCfg<8, 3, 1024>, true" -c 1 python tools/k6_bench.py --iters 2
"""
import argparse
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gib", type=float, default=4.0)
    p.add_argument("--regions", type=int, default=2)
    p.add_argument("--iters", type=int, default=5)
    a = p.parse_args()
    torch.cuda.set_device(0)
    ctx = kc.Context(0)
    n = int(a.gib * 2**30)
    vas = [ctx.alloc(n) for _ in range(a.regions)]
    g = torch.Generator(device="cuda").manual_seed(synth.seed(4, 66))
    for va in vas:
        v = synth.dev_view(va, n)
        for o in range(0, n, 1 << 30):
            k = min(1 << 30, n - o)
            v[o:o + k].copy_(torch.randint(0, 256, (k,), dtype=torch.uint8, device="cuda", generator=g))
    torch.cuda.synchronize()
    total = n * a.regions
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    disp = dict(image=image, mangled="kc_fixture_axpy_u32", grid=(1, 1, 1), block=(256, 1, 1),
                kernarg=struct.pack("<QQII", vas[0], vas[0] + 4096, 256, 3), regions=[(va, n) for va in vas])
    times = []
    snap = None
    for _ in range(a.iters):
        if snap is not None:
            snap.free()
        snap, rep = ctx.capture_dev(**disp)
        times.append(rep["t_hash_pre_s"])
    best = min(times)
    for va in vas:
        ctx.free(va)
    r, rst = ctx.restore_dev(snap)
    out = {"bytes": total, "k6_capture_ms": [1e3 * t for t in times],
           "k6_capture_traffic_gbs_best": 2 * total / best / 1e9,
           "restore_copy_in_verify_ms": 1e3 * rst["t_h2d_s"],
           "restore_traffic_gbs": 2 * total / rst["t_h2d_s"] / 1e9, "verify_mismatch": rst["verify_mismatch_chunks"]}
    print(json.dumps(out))
    r.release()
    snap.free()
    ctx.close()


if __name__ == "__main__":
    main()
