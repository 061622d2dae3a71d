"""Measure K1 variants (KC_K1_VARIANT) on resident data larger than L2.
    python tools/k1_variants.py            # all variants, one subprocess each
"""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "one":
    import numpy as np
    import torch
    from paper_2605_03208_b200 import kc
    ctx = kc.Context(0)
    res = {}
    g = torch.Generator(device="cuda").manual_seed(1)
    for name, sizes in [("1x8GiB", [8 << 30]), ("c4like", [692060160] * 8 + [346030080] * 8 + [4096] * 8 +
                                                       [int(x) for x in np.random.default_rng(0).integers(65536, 256 << 20, 40)])]:
        bufs = [torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g) for n in sizes]
        regions = sorted((b.data_ptr(), b.numel()) for b in bufs)
        C = kc.count_chunks(regions)
        out = torch.zeros(C, dtype=torch.int64, device="cuda")
        nbytes = sum(sizes)
        for _ in range(3):
            ctx.hash(regions, out.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        it = 10
        for _ in range(it):
            ctx.hash(regions, out.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        res[name] = {"ms": ms, "gbs": nbytes / ms / 1e6, "checksum": int(out.sum().item()) & 0xFFFFFFFFFFFF}
        del bufs
        torch.cuda.empty_cache()
    print(json.dumps(res))
else:
    names = {0: "cp.async 64ch x3 x1K (default)", 1: "tma-bulk 64 slots x3 x1K", 2: "tma-bulk 32 slots x3 x2K",
             3: "cp.async 128ch x3 x512"}
    base = None
    only = [int(x) for x in os.environ.get("ONLY", "").split(",") if x]
    for v, n in names.items():
        if only and v not in only:
            continue
        env = dict(os.environ, KC_K1_VARIANT=str(v))
        out = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True)
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            print(v, n, "FAILED", out.stderr[-400:])
            continue
        if base is None:
            base = {k: x["checksum"] for k, x in r.items()}
        same = all(r[k]["checksum"] == base[k] for k in r)
        print(f"{v} {n:22s} " + "  ".join(f"{k}: {x['gbs']:7.0f} GB/s ({x['ms']:.3f} ms)" for k, x in r.items()) +
              ("" if same else "  CHECKSUM MISMATCH"), flush=True)
