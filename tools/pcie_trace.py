"""PCIe evidence for A5 (D2H capture) and A6 (H2D restore): a CUPTI activity trace of
the copies the library issues, recorded with torch.profiler (Kineto = CUPTI; nsys is
not in this image).  The c4 pool (30,074,000,000 B, 185 regions) is captured into a
pinned host arena (kc_capture_host, PRE_W), the live regions are freed, and the
snapshot is restored at the same VAs (kc_restore_dev: H2D copy-in + K1 verify),
replayed and validated.  Writes a chrome trace and a per-direction summary:
bytes, copy count, busy time (union of copy intervals), span, and GB/s against the
measured pinned peak.
    python tools/pcie_trace.py [--out-dir profiles] [--tag r2]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def union_us(iv):
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in sorted(iv):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def summarize(trace, peak, head=()):
    """Per direction: all copies (count, bytes, busy time = union of intervals) and the
    snapshot stream (copies of >= 16 MiB: bytes over first-to-last span, against the
    measured pinned peak and the 64 GB/s spec)."""
    ev = json.load(open(trace))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    rows = {}
    for e in ev:
        if e.get("cat") not in ("gpu_memcpy", "Memcpy") or "dur" not in e:
            continue
        name = e.get("name", "")
        kind = "D2H" if "DtoH" in name else ("H2D" if "HtoD" in name else ("D2D" if "DtoD" in name else name))
        r_ = rows.setdefault(kind, [])
        r_.append((float(e["ts"]), float(e["ts"]) + float(e["dur"]), int(e.get("args", {}).get("bytes", 0) or 0)))
    out = list(head) + [
        f"# measured pinned peak (best of 5 x 1 GiB): D2H {peak['d2h_gbs']:.1f} GB/s, H2D {peak['h2d_gbs']:.1f} GB/s; "
        "PCIe Gen5 x16 spec 64 GB/s per direction",
        "# all = every copy (busy = union of intervals); stream = the copies of >= 16 MiB (the region pieces), "
        "bytes over first-to-last span",
        f"{'dir':4s} {'copies':>6s} {'bytes':>16s} {'busy s':>7s} | {'stream':>6s} {'bytes':>16s} {'span s':>7s} "
        f"{'GB/s':>6s} {'of meas.':>8s} {'of 64':>6s}"]
    for kind, r_ in sorted(rows.items()):
        busy = union_us([(s, e) for s, e, _ in r_]) * 1e-6
        big = [x for x in r_ if x[2] >= 16 << 20]
        nb = sum(x[2] for x in big)
        span = (max(x[1] for x in big) - min(x[0] for x in big)) * 1e-6 if big else 0.0
        gbs = nb / span / 1e9 if span else 0.0
        pk = peak["d2h_gbs"] if kind == "D2H" else peak["h2d_gbs"] if kind == "H2D" else None
        out.append(f"{kind:4s} {len(r_):6d} {sum(x[2] for x in r_):16,d} {busy:7.3f} | {len(big):6d} {nb:16,d} "
                   f"{span:7.3f} {gbs:6.1f} {gbs / pk if pk else 0:8.2f} {gbs / 64:6.2f}")
    return "\n".join(out)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out"))
    p.add_argument("--tag", default="r2")
    p.add_argument("--summarize", default=None, help="re-summarize an existing trace (no GPU): TRACE D2H_PEAK H2D_PEAK")
    a, rest = p.parse_known_args()
    if a.summarize:
        print(summarize(a.summarize, {"d2h_gbs": float(rest[0]), "h2d_gbs": float(rest[1])}))
        return
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import synth
    from paper_2605_03208_b200 import kc

    torch.cuda.set_device(0)
    ctx = kc.Context(0)
    pool = bench.Pool(ctx, 0, 1, 0, lambda *x: None)
    peak = bench.pcie_peak(lambda *x: None)
    regions = list(pool.regions)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    warps = synth.C4_T * 2816
    disp = dict(image=image, mangled="kc_fixture_moe_gemv", grid=((warps * 32 + 255) // 256, 1, 1),
                block=(256, 1, 1), kernarg=pool.kernarg, regions=regions, mode=kc.KC_MODE_PRE_W)
    ctx.host_arena_reserve(pool.bytes + 256 * len(regions))
    ys = [s for s in pool.specs if s.name == "y"][0]
    synth.dev_view(pool.va["y"], ys.size).zero_()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        snap, cap = ctx.capture_host(**disp)
        t1 = time.perf_counter()
        for s in pool.specs:
            ctx.free(pool.va[s.name])
        t2 = time.perf_counter()
        r, rst = ctx.restore_dev(snap)
        t3 = time.perf_counter()
        ctx.replay(r)
        reps, unexpected = ctx.validate(r)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
    ok = all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0 and rst["verify_mismatch_chunks"] == 0
    os.makedirs(a.out_dir, exist_ok=True)
    trace = os.path.join(a.out_dir, f"{a.tag}_pcie_trace.json")
    prof.export_chrome_trace(trace)
    head = [f"# CUPTI activity trace (torch.profiler / Kineto) of kc_capture_host + kc_restore_dev on the c4 pool "
            f"({pool.bytes:,} B, {len(regions)} regions), one B200; chrome trace: {os.path.basename(trace)}",
            f"# wall: capture {t1 - t0:.3f} s, restore {t3 - t2:.3f} s, replay + validate {t4 - t3:.3f} s; "
            f"bit-exact {ok}; library stage times: capture copy {cap['t_d2h_s']:.3f} s, restore copy-in "
            f"{rst['t_h2d_s']:.3f} s"]
    txt = summarize(trace, peak, head)
    print(txt)
    open(os.path.join(a.out_dir, f"{a.tag}_pcie_trace.txt"), "w").write(txt + "\n")
    r.release()
    snap.free()
    ctx.host_arena_reserve(0)


if __name__ == "__main__":
    main()
