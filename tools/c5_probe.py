"""c5 cells through the prepared plans, a launch target for ncu (per-kernel times):
    ncu --metrics gpu__time_duration.sum -k regex:"k1_|k2_" python tools/c5_probe.py 65536 1000"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench_configs as bc  # noqa: E402
import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402

S, n = int(sys.argv[1]), int(sys.argv[2])
ctx = kc.Context(0)
timer = bc.Timer(torch, 3)
g = torch.Generator(device="cuda").manual_seed(synth.seed(5))
res, _, keep = bc.c5_cell(torch, ctx, timer, S, n, 6545.3, g)
print(S, n, "K1", round(res["K1"]["gbs"]), round(res["K1"]["ms"] * 1e3, 1), "us", "K2", round(res["K2"]["gbs"]),
      round(res["K2"]["ms"] * 1e3, 1), "us", res["k2_found_every_flip"])
