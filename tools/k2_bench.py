"""K2 microbenchmark: identical and c3-planted pairs resident in HBM (> L2).
    python tools/k2_bench.py            # every KC_K2_VARIANT, one subprocess each
"""
import json
import os
import subprocess
import sys

if len(sys.argv) == 1:
    names = {0: "512 thr x1 CTA, 2 vec (default)"}
    for v, n in names.items():
        out = subprocess.run([sys.executable, __file__, "one"], env=dict(os.environ, KC_K2_VARIANT=str(v)),
                             capture_output=True, text=True)
        lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
        print(f"variant {v} ({n}):", " | ".join(f"{ln.split()[0]} {json.loads(ln.split(' ', 1)[1])['gbs']:.0f} GB/s"
                                                  for ln in lines) or out.stderr[-300:], flush=True)
    sys.exit(0)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402

ctx = kc.Context(0)
g = torch.Generator(device="cuda").manual_seed(3)
res = {}
n = 2 * 2**30  # elements of bf16 per buffer: 4 GiB
cases = ["identical_bf16", "c3_planted_bf16", "c3_planted_f16", "identical_bytes"]
if os.environ.get("KC_K2_CASES"):
    cases = os.environ["KC_K2_CASES"].split(",")
for name in cases:
    tdt = torch.float16 if "f16" in name and "bf16" not in name else torch.bfloat16
    ref = (torch.randn(n // 2, device="cuda", generator=g) * 0.5).to(tdt)
    act = ref.clone()
    if "planted" in name:
        synth.plant_c3(ref.view(torch.int16), act.view(torch.int16), "f16" if tdt == torch.float16 else "bf16",
                       synth.C3_MISMATCH_P, g)
    dt = "bytes" if "bytes" in name else ("f16" if tdt == torch.float16 else "bf16")
    nb = ref.numel() * 2
    bufs = [(ref.data_ptr(), act.data_ptr(), nb, dt)]
    reps = torch.zeros(15, dtype=torch.int64, device="cuda")
    for _ in range(3):
        ctx.diff_async(bufs, 1, [nb], reps.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 10
    e0.record()
    for _ in range(it):
        ctx.diff_async(bufs, 1, [nb], reps.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    res[name] = {"ms": ms, "gbs": 2 * nb / ms / 1e6, "differing_bytes": int(reps[3].item())}
    print(name, json.dumps(res[name]), flush=True)
    del ref, act
    torch.cuda.empty_cache()
