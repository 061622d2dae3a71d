"""Worker for test_gpu_diff.py::test_periodic_flush_path: K2 over every dtype with
the lane accumulators flushed every KC_K2_FLUSH_UNITS units (set by the test in
this process's environment before the library loads); the reports and bitmaps
must equal the oracle's O4.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402
from test_gpu_diff import ALL_DT, FIELDS, _dev, _pair_host  # noqa: E402

ctx = kc.Context(0)
bad = []
keep = []
bufs, exps = [], []
for i, name in enumerate(ALL_DT):
    dt = kc.DT[name]
    es = oracle.ELEM_SIZE[dt]
    n = 7 * 65536 // es + 13      # 7 chunks + a ragged tail: 28+ K2 units of 16 KiB
    r, a = _pair_host(dt, n, 91 + i, oracle, density=0.02)
    dr, pr = _dev(torch, r)
    da, pa = _dev(torch, a)
    keep += [dr, da]
    bufs.append((pr, pa, r.size, name))
    exps.append(oracle.diff(r, a, dt))
torch.cuda.synchronize()
reps, bms = ctx.diff(bufs)
for name, g, e, bm in zip(ALL_DT, reps, exps, bms):
    for f in FIELDS:
        gv, ev = g[f], e.report[f]
        if not (gv == ev or (isinstance(ev, float) and np.isnan(gv) and np.isnan(ev))):
            bad.append(f"{name} {f}: gpu {gv!r} oracle {ev!r}")
    if [int(x) for x in bm] != [int(x) for x in e.bitmap]:
        bad.append(f"{name} bitmap")
print(json.dumps({"flush_units": os.environ.get("KC_K2_FLUSH_UNITS"), "bad": bad,
                  "differing_elems": [r["differing_elems"] for r in reps]}))
ctx.close()
