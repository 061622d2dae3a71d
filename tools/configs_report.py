"""Per-config measurements for BASELINE.json configs c1-c3 (c4 is bench.py, c5 is
tools/sweep_c5.py), SURVEY.md 8(d) D.3 "Reported" column:
  c1  capture -> restore -> replay -> validate latency per stage (device snapshot), K1 time
  c2  the same, plus K1 GB/s over the 152 MiB snapshot (L2 flushed)
  c3  per dtype: K2 GB/s over the Q/K/V/O pairs (4 GiB read), K1 GB/s over the 2 GiB
      reference set; report summaries at (1e-8, 1e-5) and (1e-3, 1e-3), equal_nan 0/1
Times: CUDA events around the API call, best of --iters, L2 flushed (512 MiB write) before each.
    python tools/configs_report.py [--out profiles/r1_configs.txt]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402

FLUSH = None


def timed(fn, iters):
    best = 1e30
    for _ in range(iters):
        FLUSH.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def closure(ctx, specs, fill, dispatch, iters, name):
    vas = {s.name: ctx.alloc(s.size) for s in specs}
    fill(vas)
    torch.cuda.synchronize()
    regions = sorted((vas[s.name], s.size) for s in specs)
    C = kc.count_chunks(regions)
    h = torch.zeros(C, dtype=torch.int64, device="cuda")
    rarr = kc.region_array(regions)
    k1_ms = timed(lambda: ctx.hash(rarr, h.data_ptr()), iters)
    total = sum(s for _, s in regions)
    t0 = time.perf_counter()
    snap, cap = ctx.capture_dev(regions=regions, **dispatch(vas))
    t1 = time.perf_counter()
    for va in vas.values():
        ctx.free(va)
    t2 = time.perf_counter()
    r, rst = ctx.restore_dev(snap)
    t3 = time.perf_counter()
    ctx.replay(r)
    t4 = time.perf_counter()
    reps, unexpected = ctx.validate(r)
    t5 = time.perf_counter()
    ok = all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0 and len(reps) > 0
    r.release()
    snap.free()
    return {"config": name, "bytes": total, "regions": len(regions), "chunks": C, "k1_ms": k1_ms,
            "k1_gbs": total / (k1_ms * 1e-3) / 1e9, "written_chunks": cap["written_chunks"],
            "capture_s": t1 - t0, "restore_s": t3 - t2, "replay_s": t4 - t3, "validate_s": t5 - t4,
            "latency_s": (t1 - t0) + (t3 - t2) + (t4 - t3) + (t5 - t4), "validated_bit_exact": ok}


def c3(ctx, kind, iters):
    n = synth.C3_BUF_BYTES // 2
    g = torch.Generator(device="cuda").manual_seed(synth.seed(3, 1))
    tdt = torch.float16 if kind == "f16" else torch.bfloat16
    refs, acts = [], []
    for name, std in (("Q", 1.0), ("K", 1.0), ("V", 1.0), ("O", 0.5)):
        r = (torch.randn(n, device="cuda", generator=g) * std).to(tdt)
        a = r.clone()
        if name == "O":
            synth.plant_c3(r.view(torch.int16), a.view(torch.int16), kind, synth.C3_MISMATCH_P, g)
        if name == "K":
            a.view(torch.uint8)[synth.C3_K_FLIP_OFFSET] ^= 1
        refs.append(r)
        acts.append(a)
    torch.cuda.synchronize()
    bufs = kc.buffer_array([kc.Buffer(r.data_ptr(), a.data_ptr(), 2 * n, kc.DT[kind], i, 0)
                            for i, (r, a) in enumerate(zip(refs, acts))])
    k2_ms = timed(lambda: ctx.diff(bufs, with_bitmaps=False), iters)
    regions = sorted((r.data_ptr(), 2 * n) for r in refs)
    h = torch.zeros(kc.count_chunks(regions), dtype=torch.int64, device="cuda")
    rarr = kc.region_array(regions)
    k1_ms = timed(lambda: ctx.hash(rarr, h.data_ptr()), iters)
    summ = {}
    for tol in ((1e-8, 1e-5), (1e-3, 1e-3)):
        for eq in (False, True):
            reps, _ = ctx.diff(bufs, atol=tol[0], rtol=tol[1], equal_nan=eq)
            o = reps[3]
            summ[f"O atol={tol[0]:g} rtol={tol[1]:g} equal_nan={int(eq)}"] = {
                k: o[k] for k in ("differing_elems", "max_ulp", "max_abs", "max_rel", "nan_ref", "nan_act",
                                  "nan_pos_mismatch", "rel_undefined", "allclose_fail", "pass")}
    reps, _ = ctx.diff(bufs)
    out = {"config": f"c3 {kind}", "k2_read_bytes": 8 * n * 2, "k2_ms": k2_ms,
           "k2_gbs": 16 * n / (k2_ms * 1e-3) / 1e9, "k1_bytes": 8 * n, "k1_ms": k1_ms,
           "k1_gbs": 8 * n / (k1_ms * 1e-3) / 1e9,
           "differing_bytes_QKVO": [x["differing_bytes"] for x in reps], "O_reports": summ}
    del refs, acts
    torch.cuda.empty_cache()
    return out


def main():
    global FLUSH
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=None)
    p.add_argument("--iters", type=int, default=5)
    a = p.parse_args()
    torch.cuda.set_device(0)
    FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ctx = kc.Context(0)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    res = []

    def fill_c1(vas):
        for spec, arr in zip(synth.C1_SPECS, synth.c1_fill(vas["nodes"])):
            synth.dev_view(vas[spec.name], arr.size).copy_(torch.from_numpy(arr))
    res.append(closure(ctx, synth.C1_SPECS, fill_c1,
                       lambda v: dict(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                                      kernarg=synth.c1_kernarg(v["heads"], v["out"], v["nodes"])), a.iters, "c1"))
    c2s = synth.c2_specs()

    def fill_c2(vas):
        gen = torch.Generator(device="cuda").manual_seed(synth.seed(2))
        for s in c2s:
            synth.fill_device(synth.dev_view(vas[s.name], s.size), s, gen)
    res.append(closure(ctx, c2s, fill_c2,
                       lambda v: dict(image=image, mangled="kc_fixture_decode_attn", grid=(32, 1, 1),
                                      block=(128, 1, 1), kernarg=synth.c2_kernarg(v)), a.iters, "c2"))
    for kind in ("f16", "bf16"):
        res.append(c3(ctx, kind, a.iters))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6545.3
    lines = [f"# tools/configs_report.py on one B200; frac = GB/s / {peak} (measured copy peak); best of {a.iters}, "
             "L2 flushed before each timed call"]
    for r in res:
        if r["config"] in ("c1", "c2"):
            lines.append(f"{r['config']}: {r['bytes']:,} B in {r['regions']} regions ({r['chunks']} chunks): K1 "
                         f"{r['k1_ms'] * 1e3:.1f} us = {r['k1_gbs']:.0f} GB/s ({r['k1_gbs'] / peak:.2f}); capture "
                         f"{r['capture_s'] * 1e3:.2f} ms, restore {r['restore_s'] * 1e3:.2f} ms, replay "
                         f"{r['replay_s'] * 1e3:.2f} ms, validate {r['validate_s'] * 1e3:.2f} ms -> "
                         f"{r['latency_s'] * 1e3:.2f} ms, |W| = {r['written_chunks']}, bit-exact "
                         f"{r['validated_bit_exact']}")
        else:
            lines.append(f"{r['config']}: K2 over Q/K/V/O pairs ({r['k2_read_bytes'] / 2**30:.0f} GiB read) "
                         f"{r['k2_ms']:.3f} ms = {r['k2_gbs']:.0f} GB/s ({r['k2_gbs'] / peak:.2f}); K1 over the "
                         f"{r['k1_bytes'] / 2**30:.0f} GiB reference set {r['k1_ms']:.3f} ms = {r['k1_gbs']:.0f} GB/s "
                         f"({r['k1_gbs'] / peak:.2f}); differing bytes Q/K/V/O {r['differing_bytes_QKVO']}")
            for k, v in r["O_reports"].items():
                lines.append(f"    {k}: " + ", ".join(f"{kk} {vv:.4g}" if isinstance(vv, float) else f"{kk} {vv}"
                                                       for kk, vv in v.items()))
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")
        json.dump(res, open(os.path.splitext(a.out)[0] + ".json", "w"), indent=1, default=float)
    ctx.close()


if __name__ == "__main__":
    main()
