"""Per-config measurements for bench.py (BASELINE.json configs c1, c2, c3, c5; c4 is
bench.py's headline step) and the oracle's CPU rates.

Every GPU number is a CUDA-event time around the public C-ABI call (kc_hash,
kc_diff_async, kc_capture_dev/host, kc_restore_dev, kc_replay, kc_validate),
best of `iters`, with L2 flushed before each timed call: a 512 MiB write, then a
512 MiB read, so the timed call finds none of its inputs in L2 AND no dirty lines
(after the write alone, the first ~126 MB the call touches also pay the write-back
of the flush's dirty lines: c2 K1 40 -> 47 us, tools/c2_k1_probe.py --flushes).
Each config's result carries GB/s and its fraction of the measured HBM peak
(MEASURED_PEAKS.json) and of the 8 TB/s spec, and -- beside it -- the CPU
oracle's hash and diff rates on a bounded sample of the same config's bytes
(copied back from the device), at 1 thread and at every host core.

The oracle is imported here only for that CPU-baseline leg (task rule 3).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SPEC_HBM_GBS = 8000.0
PIECE = 4 << 20             # oracle work unit: 4 MiB (64 chunks), chunk- and element-aligned
T1_BYTES = 32 << 20         # the 1-thread rates use the first 32 MiB of a sample (bounded CPU time)


# ------------------------------------------------------------------ host + oracle rates
def host_info() -> dict:
    """nproc, lscpu model name, sockets and NUMA nodes."""
    out = {"nproc": os.cpu_count() or 1}
    try:
        import subprocess
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in txt.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                out["model"] = v
            elif k == "Socket(s)":
                out["sockets"] = int(v) if v.isdigit() else v
            elif k == "NUMA node(s)":
                out["numa_nodes"] = int(v) if v.isdigit() else v
    except Exception as ex:  # reported, never hidden
        out["lscpu_error"] = repr(ex)[:120]
    return out


def _pieces(pairs):
    """(ref, act, dtype) host byte arrays -> 16 MiB pieces (whole chunks, whole elements)."""
    out = []
    for r, a, dt in pairs:
        for o in range(0, r.size, PIECE):
            out.append((r[o:o + PIECE], a[o:o + PIECE], dt))
    return out


def oracle_rates(pairs, threads: int, min_seconds: float = 1.0, max_bytes: int | None = None) -> dict:
    """The oracle as it stands on `threads` host threads over (ref, act, dtype) pairs:
    hash GB/s = act bytes hashed (O2 chunk manifest) per second; diff GB/s = ref + act
    bytes read by the O4 report per second.  Work repeats until min_seconds each;
    max_bytes keeps only the first pieces of the sample."""
    import oracle
    oracle.build()
    pcs = _pieces(pairs)
    if max_bytes is not None:
        keep, acc = [], 0
        for pc in pcs:
            if acc >= max_bytes:
                break
            keep.append(pc)
            acc += pc[1].size
        pcs = keep
    n = sum(a.size for _, a, _ in pcs)
    res = {"threads": threads, "bytes": n}
    with ThreadPoolExecutor(threads) as ex:
        for key, fn, mult in (("hash_gbs", lambda p: oracle.chunk_hashes(p[1]), 1),
                              ("diff_gbs", lambda p: oracle.diff(p[0], p[1], p[2], with_bitmap=True), 2)):
            passes = 0
            t0 = time.perf_counter()
            while True:
                list(ex.map(fn, pcs))
                passes += 1
                if time.perf_counter() - t0 >= min_seconds:
                    break
            dt = time.perf_counter() - t0
            res[key] = mult * n * passes / dt / 1e9
            res[key.replace("gbs", "s")] = dt
    # the metric's step mix (2 hashes of N + a diff reading 2N): 4N / (2N/H + 2N/D)
    H, D = res["hash_gbs"], res["diff_gbs"]
    res["step_mix_gbs"] = 2 * H * D / (H + D)
    return res


def oracle_both(pairs, min_seconds: float, nproc: int | None = None) -> dict:
    """1 thread (on the sample's first T1_BYTES) and every host core (the whole sample)."""
    nproc = nproc or (os.cpu_count() or 1)
    return {"t1": oracle_rates(pairs, 1, min_seconds, T1_BYTES), "all_cores": oracle_rates(pairs, nproc, min_seconds)}


def sample_pairs(torch, pairs_dev, max_bytes: int):
    """Copy up to max_bytes of (ref_va, act_va, nbytes, oracle dtype) device pairs to the host,
    taking the head of every pair in turn (chunk-aligned), so every region kind is sampled."""
    import synth
    if not pairs_dev:
        return []
    per = max(65536, (max_bytes // len(pairs_dev)) // 65536 * 65536)
    out, total = [], 0
    for r, a, n, dt in pairs_dev:
        k = min(n, per)
        if total + k > max_bytes and out:
            break
        out.append((synth.dev_view(r, k).cpu().numpy().copy(), synth.dev_view(a, k).cpu().numpy().copy(), dt))
        total += k
    return out


def frac(gbs: float, peak: float) -> dict:
    return {"gbs": gbs, "frac": gbs / peak, "frac_of_spec_8000": gbs / SPEC_HBM_GBS}


# ------------------------------------------------------------------ timing helpers
class Timer:
    def __init__(self, torch, iters: int):
        self.torch, self.iters = torch, iters
        self.flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        self.flush_r = torch.zeros(64 << 20, dtype=torch.int64, device="cuda")  # 512 MiB, read back
        self.acc = torch.zeros((), dtype=torch.int64, device="cuda")

    def flush_l2(self, i: int) -> None:
        self.flush.fill_(i & 0xFF)                                 # write > L2: evicts every input line
        self.torch.sum(self.flush_r, dim=0, out=self.acc)          # read > L2: evicts the dirty flush lines

    def best_ms(self, fn) -> float:
        torch = self.torch
        best = 1e30
        for i in range(self.iters + 1):
            self.flush_l2(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i:   # the first call warms the plan caches
                best = min(best, e0.elapsed_time(e1))
        return best


# ------------------------------------------------------------------ c1 / c2: the closure
def closure(torch, ctx, timer, specs, fill, dispatch, name, peak, host=False, outputs=()):
    """K1 over the snapshot, then capture (device or pinned-host sink) -> free -> restore
    at the same VAs -> replay -> validate, each stage timed (wall clock around the call).
    `outputs` (region names) are zeroed before each capture, so the dispatch writes
    chunks (W != {}) in every cycle, also when the previous cycle's replay left its
    output in place."""
    import synth
    from paper_2605_03208_b200 import kc
    vas = {s.name: ctx.alloc(s.size) for s in specs}
    fill(vas)
    torch.cuda.synchronize()
    regions = sorted((vas[s.name], s.size) for s in specs)
    C = kc.count_chunks(regions)
    h = torch.zeros(C, dtype=torch.int64, device="cuda")
    rarr = kc.region_array(regions)
    k1_ms = timer.best_ms(lambda: ctx.hash(rarr, h.data_ptr()))
    total = sum(s for _, s in regions)
    dtype_of = {vas[s.name]: s.dtype for s in specs}
    stages = {}
    live = None   # the restored handle that holds the regions after a cycle (None: ctx.alloc'd)
    # one untimed device cycle first: the first capture / restore of a process pays
    # lazy module loading and arena setup (reported by bench.py's capture_replay
    # "cold" cycle), not what a resident tool pays per iteration
    for sink in (("warmup", "device", "host_pinned") if host else ("warmup", "device")):
        for o in outputs:
            synth.dev_view(vas[o], next(sp.size for sp in specs if sp.name == o)).zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        snap, cap = (ctx.capture_host if sink == "host_pinned" else ctx.capture_dev)(regions=regions, **dispatch(vas))
        t1 = time.perf_counter()
        if live is None:
            for va in vas.values():
                ctx.free(va)
        else:
            live.release()
        t2 = time.perf_counter()
        r, rst = ctx.restore_dev(snap)
        t3 = time.perf_counter()
        ctx.replay(r)
        t4 = time.perf_counter()
        reps, unexpected = ctx.validate(r)
        t5 = time.perf_counter()
        ok = all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0 and len(reps) > 0 \
            and rst["verify_mismatch_chunks"] == 0
        same = sorted((x.base, x.size) for x in r.regions()) == regions
        stages[sink] = {"capture_s": t1 - t0, "restore_s": t3 - t2, "replay_s": t4 - t3, "validate_s": t5 - t4,
                        "latency_s": (t1 - t0) + (t3 - t2) + (t4 - t3) + (t5 - t4), "validated_bit_exact": bool(ok),
                        "same_vas": bool(same), "written_chunks": cap["written_chunks"],
                        "capture_copy_gbs": (cap["d2h_bytes"] or total) / max(cap["t_d2h_s"], 1e-9) / 1e9,
                        "restore_copy_gbs": rst["h2d_bytes"] / max(rst["t_h2d_s"], 1e-9) / 1e9}
        snap.free()
        live = r
    stages.pop("warmup")
    # identical (captured, replayed) pairs: what the closure validated; the caller samples
    # them for the oracle, then releases `live`
    pairs_dev = [(b, b, n, dtype_of[b]) for b, n in regions]
    return {"config": name, "bytes": total, "regions": len(regions), "chunks": C,
            "K1": dict(frac(total / (k1_ms * 1e-3) / 1e9, peak), ms=k1_ms), "closure": stages}, pairs_dev, live


def c3(torch, ctx, timer, kind, peak):
    """c3: Q/K/V/O reference + actual sets (2 GiB each), O planted at the paper's 11.3%
    ULP-level mismatch density (+ NaN/Inf/signed-zero specials), K with one flipped byte.
    K2 over the 4 pairs (4 GiB read), K1 over the 2 GiB reference set, O's report."""
    import synth
    from paper_2605_03208_b200 import kc
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
    bufs = [(r.data_ptr(), a.data_ptr(), 2 * n, kind) for r, a in zip(refs, acts)]
    reps_d = torch.zeros(4 * 15, dtype=torch.int64, device="cuda")
    k2_ms = timer.best_ms(lambda: ctx.diff_async(bufs, 4, [2 * n] * 4, reps_d.data_ptr()))
    regions = sorted((r.data_ptr(), 2 * n) for r in refs)
    h = torch.zeros(kc.count_chunks(regions), dtype=torch.int64, device="cuda")
    rarr = kc.region_array(regions)
    k1_ms = timer.best_ms(lambda: ctx.hash(rarr, h.data_ptr()))
    reps, _ = ctx.diff(bufs)
    o = reps[3]
    out = {"config": f"c3 {kind}", "K2": dict(frac(16 * n / (k2_ms * 1e-3) / 1e9, peak), ms=k2_ms,
                                               read_bytes=16 * n),
           "K1": dict(frac(8 * n / (k1_ms * 1e-3) / 1e9, peak), ms=k1_ms, bytes=8 * n),
           "differing_bytes_QKVO": [x["differing_bytes"] for x in reps],
           "O_report": {k: o[k] for k in ("differing_elems", "max_ulp", "max_abs", "max_rel", "nan_ref", "nan_act",
                                          "nan_pos_mismatch", "rel_undefined", "allclose_fail", "pass")},
           "O_mismatch_fraction": o["differing_elems"] / o["n_elems"]}
    code = {"f16": 9, "bf16": 10}[kind]
    pairs_dev = [(r.data_ptr(), a.data_ptr(), 2 * n, code) for r, a in zip(refs, acts)]
    return out, pairs_dev, (refs, acts)


C5_BENCH_CELLS = [(4096, 100000), (65536, 1000), (65536, 10000), (2**20, 1000), (16 * 2**20, 100),
                  (256 * 2**20, 100)]


def c5_cell(torch, ctx, timer, S, n, peak, g):
    """One c5 cell: n regions of S + U[0, 4096) bytes, uniform random bytes, one flipped
    byte per region in the actual copy; K1 over the n regions, K2 (bytes) over n pairs."""
    import ctypes
    import synth
    from paper_2605_03208_b200 import kc
    sizes = synth.c5_sizes(S, n, jitter=True)
    offs = np.concatenate([[0], np.cumsum((sizes + 255) // 256 * 256)])
    total = int(offs[-1])
    ref = torch.empty(total, dtype=torch.uint8, device="cuda")
    for o in range(0, total, 1 << 30):
        k = min(1 << 30, total - o)
        ref[o:o + k].copy_(torch.randint(0, 256, (k,), dtype=torch.uint8, device="cuda", generator=g))
    act = ref.clone()
    act[torch.from_numpy(offs[:-1] + (sizes // 2)).cuda()] ^= 1
    base = ref.data_ptr()
    regions = [(base + int(o), int(s)) for o, s in zip(offs[:-1], sizes)]
    C = kc.count_chunks(regions)
    h = torch.zeros(max(1, C), dtype=torch.int64, device="cuda")
    bufs = kc.buffer_array([kc.Buffer(base + int(o), act.data_ptr() + int(o), int(s), 0, i, 0)
                            for i, (o, s) in enumerate(zip(offs[:-1], sizes))])
    reps = torch.zeros(n * 15, dtype=torch.int64, device="cuda")
    nb = (ctypes.c_uint64 * n)(*[int(s) for s in sizes])
    rarr = kc.region_array(regions)
    # per call (kc_hash / kc_diff_async: the region / buffer list re-checked on the host
    # every call) and prepared (kc_hash_plan / kc_diff_plan: the launches alone)
    k1c_ms = timer.best_ms(lambda: ctx.hash(rarr, h.data_ptr(), n=n))
    k2c_ms = timer.best_ms(lambda: ctx.diff_async(bufs, n, nb, reps.data_ptr()))
    found = int(reps.view(n, 15)[:, 3].sum().item()) == n
    hp = ctx.hash_plan(regions)
    dp = ctx.diff_plan(bufs, n, [int(x) for x in sizes])
    h2 = torch.zeros_like(h)
    k1_ms = timer.best_ms(lambda: hp.run(h2.data_ptr()))
    reps.zero_()
    k2_ms = timer.best_ms(lambda: dp.run(reps.data_ptr()))
    found = found and int(reps.view(n, 15)[:, 3].sum().item()) == n and bool(torch.equal(h, h2))
    hp.close()
    dp.close()
    nbytes = int(sizes.sum())
    out = {"S": S, "n": n, "bytes": nbytes, "chunks": C,
           "K1": dict(frac(nbytes / (k1_ms * 1e-3) / 1e9, peak), ms=k1_ms, api="kc_hash_plan_run"),
           "K2": dict(frac(2 * nbytes / (k2_ms * 1e-3) / 1e9, peak), ms=k2_ms, api="kc_diff_plan_run"),
           "K1_per_call": dict(frac(nbytes / (k1c_ms * 1e-3) / 1e9, peak), ms=k1c_ms, api="kc_hash"),
           "K2_per_call": dict(frac(2 * nbytes / (k2c_ms * 1e-3) / 1e9, peak), ms=k2c_ms, api="kc_diff_async"),
           "k2_found_every_flip": found}
    pairs_dev = [(base + int(o), act.data_ptr() + int(o), int(s), 0) for o, s in zip(offs[:-1], sizes)]
    return out, pairs_dev, (ref, act)
