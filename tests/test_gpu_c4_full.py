"""Parity at BASELINE.json's full size (config c4: the 30,074,000,000-byte MoE
pool, 185 regions) in the launch configuration bench.py times: the same Pool,
the same kc_hash / kc_diff_async / kc_hash_diff_async calls.

Full size, every output:
* K1: all 458,973 chunk hashes of the 30 GB manifest recomputed by the
  oracle (O2) from the chunk bytes, region by region (each region copied to
  pinned host memory, hashed on every host core); every region digest and
  the snapshot digest recomputed from the oracle's own manifest;
* K2 / K5: every region's report and bitmap against oracle.diff (O4) over
  the region's full reference and actual bytes (the reference copy carries
  seeded plants: bf16 +-k ULP, a NaN, a pointer-table entry).

Sampled (fast, kept as a first failure signal):
* K1: ~600 chunk hashes (the first and last chunk of every region, plus a
  seeded sample) recomputed from the chunk bytes; region digests and the
  snapshot digest recomputed from the manifest;
* K2 / K5: the reference copy gets seeded plants (bf16 +-k ULP, a NaN, a
  pointer-table entry) in a few chunks; every other chunk is bit-identical
  and contributes nothing, so each region's report equals the oracle's
  report over its planted chunks (sums and maxima), with the size-derived
  fields recomputed from the region size; bitmaps likewise.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]

CH = 65536
FIELDS = ["differing_bytes", "differing_elems", "max_ulp", "max_abs", "max_rel", "nan_ref", "nan_act",
          "nan_pos_mismatch", "rel_undefined", "allclose_fail"]


@pytest.fixture(scope="module")
def pool():
    import torch
    import bench
    import oracle
    from paper_2605_03208_b200 import build, kc
    build.build()
    oracle.build()
    ctx = kc.Context(0)
    p = bench.Pool(ctx, 0, 1, 0, lambda *a: None)
    yield torch, kc, ctx, oracle, p
    ctx.close()


def _chunk(torch, va, off, n):
    import synth
    return synth.dev_view(va + off, n).cpu().numpy().copy()


def test_c4_manifest_and_digests_sampled(pool):
    torch, kc, ctx, orc, p = pool
    C = kc.count_chunks(p.regions)
    assert C == 458973 and p.bytes == 30_074_000_000
    d_h = torch.zeros(C, dtype=torch.int64, device="cuda")
    nreg = len(p.regions)
    d_dig = torch.zeros(nreg + 1, dtype=torch.int64, device="cuda")
    ctx.hash(p.regions, d_h.data_ptr(), d_dig.data_ptr(), d_dig.data_ptr() + 8 * nreg)
    torch.cuda.synchronize()
    h = d_h.cpu().numpy().view(np.uint64)
    dig = d_dig.cpu().numpy().view(np.uint64)
    rng = np.random.default_rng(4)
    off = 0
    picks = []
    for j, (base, size) in enumerate(p.regions):
        nc = (size + CH - 1) // CH
        picks += [(j, off, base, size, 0), (j, off, base, size, nc - 1)]
        off += nc
    starts = np.cumsum([0] + [(s + CH - 1) // CH for _, s in p.regions])
    for g in rng.integers(0, C, size=256):
        j = int(np.searchsorted(starts, g, side="right") - 1)
        base, size = p.regions[j]
        picks.append((j, int(starts[j]), base, size, int(g - starts[j])))
    for j, c0, base, size, k in picks:
        n = min(CH, size - k * CH)
        data = _chunk(torch, base, k * CH, n)
        assert int(orc.chunk_hashes(data)[0]) == int(h[c0 + k]), f"region {j} chunk {k}"
    # digests from the (sample-verified) manifest
    for j, (base, size) in enumerate(p.regions):
        nc = (size + CH - 1) // CH
        assert orc.region_digest(h[starts[j]:starts[j] + nc]) == int(dig[j]), f"region {j} digest"
    S = orc.snapshot_digest([b for b, _ in p.regions], [s for _, s in p.regions], [int(x) for x in dig[:nreg]])
    assert S == int(dig[nreg])


def _host_regions(torch, vas_sizes, depth: int = 3):
    """Yield (index, host uint8 array) for each (va, size), copying region i+1..i+depth
    device->host on a side stream while the caller works on region i."""
    import synth
    stream = torch.cuda.Stream()
    pend = []
    it = iter(enumerate(vas_sizes))

    def issue():
        try:
            i, (va, n) = next(it)
        except StopIteration:
            return
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        with torch.cuda.stream(stream):
            h.copy_(synth.dev_view(va, n), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        pend.append((i, h, ev))
    for _ in range(depth):
        issue()
    while pend:
        i, h, ev = pend.pop(0)
        ev.synchronize()
        issue()
        yield i, h.numpy()


def test_c4_full_manifest_every_chunk_vs_oracle(pool):
    """All 458,973 chunk hashes of the 30 GB snapshot equal the oracle's (O2), and the
    region digests and snapshot digest equal the oracle's computed from its OWN manifest."""
    torch, kc, ctx, orc, p = pool
    C = kc.count_chunks(p.regions)
    nreg = len(p.regions)
    d_h = torch.zeros(C, dtype=torch.int64, device="cuda")
    d_dig = torch.zeros(nreg + 1, dtype=torch.int64, device="cuda")
    ctx.hash(p.regions, d_h.data_ptr(), d_dig.data_ptr(), d_dig.data_ptr() + 8 * nreg)
    torch.cuda.synchronize()
    h = d_h.cpu().numpy().view(np.uint64)
    dig = d_dig.cpu().numpy().view(np.uint64)
    threads = max(1, os.cpu_count() or 1)
    starts = np.cumsum([0] + [(s + CH - 1) // CH for _, s in p.regions])
    odig, checked = [], 0
    for j, data in _host_regions(torch, p.regions):
        eh = orc.chunk_hashes(data, threads=threads)
        got = h[starts[j]:starts[j + 1]]
        bad = np.nonzero(eh != got)[0]
        assert bad.size == 0, f"region {j}: {bad.size} chunk hashes differ, first chunk {int(bad[0])}"
        checked += eh.size
        odig.append(orc.region_digest(eh))
    assert checked == C == 458973
    assert odig == [int(x) for x in dig[:nreg]], "region digests != oracle"
    S = orc.snapshot_digest([b for b, _ in p.regions], [s for _, s in p.regions], odig)
    assert S == int(dig[nreg]), "snapshot digest != oracle"


def _plant(torch, p, rng):
    """Seeded plants in the REFERENCE copy; returns {region index: sorted planted chunk list}."""
    import synth
    planted = {}
    bf16 = [j for j, s in enumerate(p.specs) if s.dtype == "bf16" and s.fill != "zero" and s.size > 4 * CH]
    for j in rng.choice(bf16, size=12, replace=False):
        s = p.specs[j]
        nc = (s.size + CH - 1) // CH
        for k in sorted(set(int(x) for x in rng.integers(0, nc, size=3))):
            n = min(CH, s.size - k * CH) // 2
            v = synth.dev_view(p.ref[s.name] + k * CH, 2 * n).view(torch.int16)
            idx = torch.from_numpy(rng.integers(0, n, size=5)).cuda()
            delta = torch.from_numpy(rng.integers(1, 17, size=5) * rng.choice([-1, 1], size=5)).to(torch.int16).cuda()
            v[idx] = v[idx] + delta
            planted.setdefault(int(j), set()).add(k)
    # a NaN in one reference element, one pointer-table entry off by 8 bytes
    j = int(bf16[0])
    synth.dev_view(p.ref[p.specs[j].name] + 2 * CH + 6, 2).view(torch.int16)[0] = 0x7FC1
    planted.setdefault(j, set()).add(2)
    pj = [j for j, s in enumerate(p.specs) if s.name.startswith("ptr_")][0]
    synth.dev_view(p.ref[p.specs[pj].name] + 40, 8).view(torch.int64)[0] += 8
    planted.setdefault(pj, set()).add(0)
    torch.cuda.synchronize()
    return {j: sorted(ks) for j, ks in planted.items()}


def _expected(torch, orc, kc, p, planted):
    """Per-region expected report fields and bitmap bit set, from the oracle over planted chunks."""
    out = {}
    for j, s in enumerate(p.specs):
        dt = kc.DT[s.dtype]
        es = orc.ELEM_SIZE[dt]
        e = {f: 0 for f in FIELDS}
        e.update(max_abs=0.0, max_rel=0.0)
        bits = set()
        if j in planted:
            rs, as_ = [], []
            for k in planted[j]:
                n = min(CH, s.size - k * CH)
                rs.append(_chunk(torch, p.ref[s.name], k * CH, n))
                as_.append(_chunk(torch, p.va[s.name], k * CH, n))
            ex = orc.diff(np.concatenate(rs), np.concatenate(as_), dt)
            for f in FIELDS:
                e[f] = ex.report[f]
            for q, k in enumerate(planted[j]):
                if (int(ex.bitmap[q // 64]) >> (q % 64)) & 1:
                    bits.add(k)
        e["nbytes"] = s.size
        e["n_elems"] = s.size // es
        e["n_chunks"] = (s.size + CH - 1) // CH
        e["percent_bytes"] = (100.0 * e["differing_bytes"]) / s.size
        e["pass"] = int(e["allclose_fail"] == 0) if s.dtype in ("f16", "bf16", "f32", "f64") else \
            int(e["differing_elems"] == 0)
        out[j] = (e, bits)
    return out


def _expected_full(torch, orc, kc, p):
    """Per-region report and bitmap bit set from oracle.diff over the WHOLE region (O4):
    reference and actual bytes streamed to the host, regions diffed in parallel."""
    out = {}
    refs = _host_regions(torch, [(p.ref[s.name], s.size) for s in p.specs], depth=2)
    acts = _host_regions(torch, [(p.va[s.name], s.size) for s in p.specs], depth=2)

    def one(j, r, a):
        s = p.specs[j]
        ex = orc.diff(r, a, kc.DT[s.dtype])
        nc = (s.size + CH - 1) // CH
        bits = {k for k in range(nc) if (int(ex.bitmap[k // 64]) >> (k % 64)) & 1}
        return j, (dict(ex.report), bits)
    with ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        futs = []
        for (j, r), (j2, a) in zip(refs, acts):
            assert j == j2
            futs.append(ex.submit(one, j, r.copy(), a.copy()))
            if len(futs) >= 16:     # bound host memory: at most ~16 regions in flight
                for f in futs[:8]:
                    jj, v = f.result()
                    out[jj] = v
                futs = futs[8:]
        for f in futs:
            jj, v = f.result()
            out[jj] = v
    return out


def _check(kc, reps_raw, bms, word0, exp, p, label):
    for j, s in enumerate(p.specs):
        got = kc.DiffReport.from_buffer_copy(reps_raw[120 * j:120 * (j + 1)]).as_dict()
        e, bits = exp[j]
        for f, v in e.items():
            g = got[f]
            assert (g == v) or (isinstance(v, float) and np.isnan(g) and np.isnan(v)), \
                f"{label} region {j} ({s.name}) {f}: gpu {g!r} expected {v!r}"
        nc = (s.size + CH - 1) // CH
        words = bms[word0[j]:word0[j] + (nc + 63) // 64]
        got_bits = {k for k in range(nc) if (int(words[k // 64]) >> (k % 64)) & 1}
        assert got_bits == bits, f"{label} region {j} bitmap"


def test_c4_k2_and_k5_reports_full_size(pool):
    torch, kc, ctx, orc, p = pool
    rng = np.random.default_rng(260503208 + 4)
    planted = _plant(torch, p, rng)
    exp = _expected(torch, orc, kc, p, planted)
    bufs, nb, word0, acc = p.diff_buffers()   # bench.py's buffers, report sizes and bitmap offsets
    assert [b.nbytes for b in bufs] == nb
    reps = torch.zeros(len(bufs) * 15, dtype=torch.int64, device="cuda")
    bms = torch.zeros(acc, dtype=torch.int64, device="cuda")
    # bench.py's K2 call
    ctx.diff_async(bufs, len(bufs), nb, reps.data_ptr(), word0, bms.data_ptr())
    torch.cuda.synchronize()
    _check(kc, reps.cpu().numpy().tobytes(), bms.cpu().numpy().view(np.uint64), word0, exp, p, "K2")
    # bench.py's fused call (F2): same reports and bitmaps, and the manifest equals K1's
    C = kc.count_chunks(p.regions)
    d_h5 = torch.zeros(C, dtype=torch.int64, device="cuda")
    d_h1 = torch.zeros(C, dtype=torch.int64, device="cuda")
    reps.zero_()
    bms.zero_()
    dirty = torch.zeros((C + 63) // 64, dtype=torch.int64, device="cuda")
    ctx.hash_diff_async(bufs, d_h5.data_ptr(), reps.data_ptr(), bms.data_ptr(), dirty.data_ptr())
    ctx.hash(p.regions, d_h1.data_ptr())
    torch.cuda.synchronize()
    _check(kc, reps.cpu().numpy().tobytes(), bms.cpu().numpy().view(np.uint64), word0, exp, p, "K5+K2")
    assert torch.equal(d_h5, d_h1)
    # every field of every region's report, and every bitmap bit, against the oracle over
    # the full 2 x 30 GB (not only the planted chunks)
    full = _expected_full(torch, orc, kc, p)
    assert len(full) == len(p.specs)
    _check(kc, reps.cpu().numpy().tobytes(), bms.cpu().numpy().view(np.uint64), word0, full, p, "K5+K2 full")
    # every planted chunk is dirty; the dirty set stays small (tails + plants)
    starts = np.cumsum([0] + [(s.size + CH - 1) // CH for s in p.specs])
    dw = dirty.cpu().numpy().view(np.uint64)
    for j, ks in planted.items():
        for k in ks:
            g = int(starts[j]) + k
            assert (int(dw[g // 64]) >> (g % 64)) & 1
    assert sum(bin(int(w)).count("1") for w in dw) < 1000
