"""Seeded randomized parity of K2 (and K5 + filtered K2, and the prepared K2 plan)
against the oracle's O4: every dtype, lengths from 1 element to several 16 KiB units
and 64 KiB chunks, mismatch densities from 0 to 100%, IEEE specials, misaligned
operands, and tolerances including 0, the numpy defaults, loose ones, atol-only and
rtol-only, with and without equal_nan.  Each case is a fresh draw from one seed, so
a failure is reproducible from its index."""
import numpy as np
import pytest

from test_gpu_diff import FIELDS, _dev, _pair_host, _same

pytestmark = pytest.mark.gpu
CH = 65536
ALL_DT = ["bytes", "u8", "i8", "u16", "i16", "u32", "i32", "u64", "i64", "f16", "bf16", "f32", "f64"]
TOLS = [(0.0, 0.0), (1e-8, 1e-5), (1e-3, 1e-3), (1e-2, 0.0), (0.0, 1e-2), (1.0, 0.5)]
DENS = [0.0, 1e-5, 1e-2, 0.113, 0.5, 1.0]


@pytest.fixture(scope="module")
def env():
    import torch
    import oracle
    from paper_2605_03208_b200 import build, kc
    build.build()
    oracle.build()
    ctx = kc.Context(0)
    yield torch, kc, ctx, oracle
    ctx.close()


def _draw(orc, i):
    rng = np.random.default_rng(260503208 + 7919 * i)
    name = ALL_DT[int(rng.integers(0, len(ALL_DT)))]
    dt = orc.DTYPE_NAMES.index(name)
    es = orc.ELEM_SIZE[dt]
    n = int(rng.choice([1, 7, 31, 33, 511, 4097, 8192 + 3, 65536 // es + 5, 300_000 // es, 3 * 65536 // es - 1]))
    density = float(rng.choice(DENS))
    specials = bool(rng.integers(0, 2))
    tol = TOLS[int(rng.integers(0, len(TOLS)))]
    eq = bool(rng.integers(0, 2))
    offs = (es * int(rng.integers(0, 4)), es * int(rng.integers(0, 4)))
    return name, dt, n, density, specials, tol, eq, offs, int(rng.integers(0, 2**31))


@pytest.mark.parametrize("block", range(10))
def test_k2_random_cases_match_oracle(env, block):
    torch, kc, ctx, orc = env
    for i in range(block * 60, block * 60 + 60):
        name, dt, n, density, specials, tol, eq, offs, seed = _draw(orc, i)
        r, a = _pair_host(dt, n, seed, orc, specials=specials, density=density)
        tr, pr = _dev(torch, r, offs[0])
        ta, pa = _dev(torch, a, offs[1])
        reps, bms = ctx.diff([(pr, pa, r.size, name)], atol=tol[0], rtol=tol[1], equal_nan=eq)
        e = orc.diff(r, a, dt, atol=tol[0], rtol=tol[1], equal_nan=eq)
        _same(reps[0], e.report, f"case {i}: {name} n={n} dens={density} tol={tol} eq={eq} offs={offs}")
        assert [int(w) for w in bms[0]] == [int(w) for w in e.bitmap], f"case {i} bitmap"


def test_k5_and_plan_random_sets_match_oracle(env):
    """Random sets of aligned pairs through the fused K5 + filtered K2 and through a
    prepared K2 plan run twice: identical reports, bitmaps and manifests to the oracle."""
    torch, kc, ctx, orc = env
    for t in range(16):
        rng = np.random.default_rng(1000 + t)
        cases = [_draw(orc, 5000 + 10 * t + k) for k in range(int(rng.integers(2, 7)))]
        keep, bufs, host = [], [], []
        for name, dt, n, density, specials, tol, eq, _o, seed in cases:
            r, a = _pair_host(dt, n, seed, orc, specials=specials, density=density)
            tr, pr = _dev(torch, r)
            ta, pa = _dev(torch, a)
            keep += [tr, ta]
            bufs.append((pr, pa, r.size, name))
            host.append((r, a, dt))
        tol, eq = cases[0][5], cases[0][6]
        nck = [orc.n_chunks(r.size) for r, _, _ in host]
        words = [(c + 63) // 64 for c in nck]
        w0 = list(np.cumsum([0] + words[:-1]))
        d_h = torch.zeros(sum(nck), dtype=torch.int64, device="cuda")
        d_rep = torch.zeros(len(bufs) * 15, dtype=torch.int64, device="cuda")
        d_bm = torch.zeros(max(1, sum(words)), dtype=torch.int64, device="cuda")
        d_dirty = torch.zeros((sum(nck) + 63) // 64 + 1, dtype=torch.int64, device="cuda")
        ctx.hash_diff_async(bufs, d_h.data_ptr(), d_rep.data_ptr(), d_bm.data_ptr(), d_dirty.data_ptr(),
                            atol=tol[0], rtol=tol[1], equal_nan=eq)
        torch.cuda.synchronize()
        exp = [orc.diff(r, a, dt, atol=tol[0], rtol=tol[1], equal_nan=eq) for r, a, dt in host]

        def check(label):
            raw, bm = d_rep.cpu().numpy().tobytes(), d_bm.cpu().numpy().view(np.uint64)
            for j, e in enumerate(exp):
                _same(kc.DiffReport.from_buffer_copy(raw[120 * j:120 * (j + 1)]).as_dict(), e.report, f"{label} {t}.{j}")
                assert [int(x) for x in bm[w0[j]:w0[j] + words[j]]] == [int(x) for x in e.bitmap], f"{label} {t}.{j}"
        check("K5+K2")
        man = np.concatenate([orc.chunk_hashes(a) for _, a, _ in host])
        assert np.array_equal(d_h.cpu().numpy().view(np.uint64), man)
        plan = ctx.diff_plan(bufs, len(bufs), [b[2] for b in bufs], w0)
        for _ in range(2):
            d_rep.fill_(-1)
            plan.run(d_rep.data_ptr(), d_bm.data_ptr(), atol=tol[0], rtol=tol[1], equal_nan=eq)
            torch.cuda.synchronize()
            check("plan")
        plan.close()


@pytest.mark.parametrize("block", range(4))
def test_k1_random_region_sets_match_oracle(env, block):
    """Random region sets (1 to 2,000 regions of 1 B to ~4 chunks, 16-byte aligned or not,
    so both the cp.async rings (large and sub-wave) and the generic path run) through
    kc_hash and a prepared plan: every chunk hash, region digest and the snapshot digest
    equal the oracle's."""
    torch, kc, ctx, orc = env
    for t in range(block * 6, block * 6 + 6):
        rng = np.random.default_rng(77 + t)
        nreg = int(rng.choice([1, 3, 40, 700, 2000]))
        sizes = [int(x) for x in rng.choice([1, 31, 32, 33, 4096, 65535, 65536, 65537, 200_000, 262_144], size=nreg)]
        sizes = [s + int(rng.integers(0, 64)) for s in sizes]
        align = 16 if rng.integers(0, 3) else 8
        offs = np.concatenate([[0], np.cumsum([(s + 255) // 256 * 256 for s in sizes])])
        buf = torch.randint(0, 256, (int(offs[-1]) + 64,), dtype=torch.uint8, device="cuda")
        shift = 0 if align == 16 else 8
        regions = [(buf.data_ptr() + int(o) + shift, s) for o, s in zip(offs[:-1], sizes)]
        C = kc.count_chunks(regions)
        h = torch.zeros(C, dtype=torch.int64, device="cuda")
        dg = torch.zeros(nreg + 1, dtype=torch.int64, device="cuda")
        ctx.hash(regions, h.data_ptr(), dg.data_ptr(), dg.data_ptr() + 8 * nreg)
        torch.cuda.synchronize()
        host = buf.cpu().numpy()
        base = buf.data_ptr()
        man = [orc.chunk_hashes(host[b - base:b - base + s]) for b, s in regions]
        assert np.array_equal(h.cpu().numpy().view(np.uint64), np.concatenate(man)), f"set {t} manifest"
        digs = [orc.region_digest(m) for m in man]
        assert [int(x) for x in dg.cpu().numpy().view(np.uint64)[:nreg]] == digs, f"set {t} digests"
        assert int(dg.cpu().numpy().view(np.uint64)[nreg]) == orc.snapshot_digest(
            [b for b, _ in regions], sizes, digs), f"set {t} snapshot digest"
        plan = ctx.hash_plan(regions)
        h2 = torch.zeros_like(h)
        plan.run(h2.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(h, h2), f"set {t} plan"
        plan.close()
