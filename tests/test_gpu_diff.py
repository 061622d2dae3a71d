"""GPU parity of K2 (fused diff) against the oracle's O4 report.

Bar (north star): bit-exact counts, bitmaps, ULP distances; max abs/rel in
fp64 with 0 relative difference (compared with ==)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CH = 65536
FIELDS = ["nbytes", "n_elems", "n_chunks", "differing_bytes", "differing_elems", "max_ulp", "max_abs", "max_rel",
          "percent_bytes", "nan_ref", "nan_act", "nan_pos_mismatch", "rel_undefined", "allclose_fail", "pass"]


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2605_03208_b200 import build, kc
    import oracle
    build.build()
    oracle.build()
    ctx = kc.Context(0)
    yield torch, kc, ctx, oracle
    ctx.close()


def _same(got, exp, ctxmsg=""):
    for f in FIELDS:
        g, e = got[f], exp[f]
        if isinstance(e, float):
            assert (g == e) or (np.isnan(g) and np.isnan(e)), f"{ctxmsg} {f}: gpu {g!r} oracle {e!r}"
        else:
            assert g == e, f"{ctxmsg} {f}: gpu {g} oracle {e}"


def _pair_host(dt, n_elems, seed, orc, specials=True, density=0.113):
    """Random typed reference + actual with planted mismatches (host numpy)."""
    rng = np.random.default_rng(seed)
    s = orc.ELEM_SIZE[dt]
    ut = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[s]
    if dt == orc.DT_F16:
        r = rng.standard_normal(n_elems).astype(np.float16).view(np.uint16)
    elif dt == orc.DT_BF16:
        r = (rng.standard_normal(n_elems).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    elif dt == orc.DT_F32:
        r = rng.standard_normal(n_elems).astype(np.float32).view(np.uint32)
    elif dt == orc.DT_F64:
        r = rng.standard_normal(n_elems).view(np.uint64)
    else:
        r = rng.integers(0, np.iinfo(ut).max, size=n_elems, dtype=ut, endpoint=True)
    r = r.copy()
    a = r.copy()
    m = rng.random(n_elems) < density
    k = np.where(rng.random(n_elems) < 0.9, 1, rng.integers(2, 17, size=n_elems))
    sg = np.where(rng.random(n_elems) < 0.5, -1, 1)
    a[m] = (a[m].astype(np.int64) + (sg * k)[m]).astype(ut)
    if specials and dt in (orc.DT_F16, orc.DT_BF16, orc.DT_F32, orc.DT_F64) and n_elems > 64:
        sign = 1 << (8 * s - 1)
        ex = {orc.DT_F16: 0x7C00, orc.DT_BF16: 0x7F80, orc.DT_F32: 0x7F800000, orc.DT_F64: 0x7FF0000000000000}[dt]
        q = ex | 1
        pos = [n_elems // 9 * j + 3 for j in range(1, 9)]
        a[pos[0]] = q
        r[pos[1]] = q; a[pos[1]] = q
        r[pos[2]] = q; a[pos[2]] = q | 2
        a[pos[3]] = ex
        r[pos[4]] = 0; a[pos[4]] = sign
        r[pos[5]] = 0; a[pos[5]] = 1
        r[pos[6]] = ex; a[pos[6]] = ex | sign
        r[pos[7]] = ex
    return r.view(np.uint8), a.view(np.uint8)


def _dev(torch, host, offset=0):
    t = torch.empty(host.size + offset + 64, dtype=torch.uint8, device="cuda")
    t[offset:offset + host.size].copy_(torch.from_numpy(host))
    return t, t.data_ptr() + offset


ALL_DT = ["bytes", "u8", "i8", "u16", "i16", "u32", "i32", "u64", "i64", "f16", "bf16", "f32", "f64"]


@pytest.mark.parametrize("dtname", ALL_DT)
@pytest.mark.parametrize("nbytes", [8, 4096, 3 * CH + 40, 700 * 1024 + 24])
def test_k2_parity_all_dtypes(env, dtname, nbytes):
    torch, kc, ctx, orc = env
    dt = orc.DTYPE_NAMES.index(dtname)
    s = orc.ELEM_SIZE[dt]
    n = nbytes // s
    r, a = _pair_host(dt, n, seed=nbytes + dt, orc=orc)
    tr, pr = _dev(torch, r)
    ta, pa = _dev(torch, a)
    for tol in [(1e-8, 1e-5, False), (1e-3, 1e-3, True)]:
        reps, bms = ctx.diff([(pr, pa, r.size, dtname)], atol=tol[0], rtol=tol[1], equal_nan=tol[2])
        exp = orc.diff(r, a, dt, atol=tol[0], rtol=tol[1], equal_nan=tol[2])
        _same(reps[0], exp.report, f"{dtname} {nbytes} {tol}")
        assert [int(w) for w in bms[0]] == [int(w) for w in exp.bitmap]


@pytest.mark.parametrize("dtname", ["bytes", "f16", "bf16", "f32", "f64", "i32"])
def test_k2_misaligned_scalar_path(env, dtname):
    torch, kc, ctx, orc = env
    dt = orc.DTYPE_NAMES.index(dtname)
    s = orc.ELEM_SIZE[dt]
    r, a = _pair_host(dt, (2 * CH + 1000) // s, seed=5 + dt, orc=orc)
    tr, pr = _dev(torch, r, offset=s)       # element-aligned, not 32-byte aligned
    ta, pa = _dev(torch, a, offset=3 * s)
    reps, bms = ctx.diff([(pr, pa, r.size, dtname)])
    exp = orc.diff(r, a, dt)
    _same(reps[0], exp.report, dtname)
    assert [int(w) for w in bms[0]] == [int(w) for w in exp.bitmap]


def _spread16(dt, n, spread, rng, orc, flip=0.3, density=0.4):
    """16-bit float pair: finite references over the whole exponent range, and
    actuals whose exponent field moves by up to `spread` (the fp32 fast path
    holds up to 13 / 16; beyond it elem_float decides), random signs and
    mantissas, zeros and subnormals."""
    eb, em = (10, 0x1F) if dt == orc.DT_F16 else (7, 0xFF)
    mant = (1 << eb) - 1
    er = rng.integers(0, em, size=n)                       # finite fields only
    r = (rng.integers(0, 2, size=n) << 15) | (er << eb) | rng.integers(0, mant + 1, size=n)
    ea = np.clip(er + rng.integers(-spread, spread + 1, size=n), 0, em - 1)
    sa = (r >> 15) ^ (rng.random(n) < flip)
    a = (sa << 15) | (ea << eb) | rng.integers(0, mant + 1, size=n)
    a = np.where(rng.random(n) < density, a, r)
    z = rng.random(n) < 0.02                               # +-0 references and actuals
    r = np.where(z, rng.integers(0, 2, size=n) << 15, r)
    return r.astype(np.uint16).view(np.uint8), a.astype(np.uint16).view(np.uint8)


@pytest.mark.parametrize("dtname", ["f16", "bf16"])
def test_k2_16bit_exponent_spread_and_tolerance_edges(env, dtname):
    """16-bit float elements take an fp32 path (DESIGN.md §7 K2) when their exponents are
    close.  Many 4 KiB buffers (one report each, so per-buffer maxima are seen),
    exponent spreads from 0 to 20 fields around the 13 / 16 limits, bf16 fields
    up to 254 (fp32 overflow of a - r), Inf/NaN in a few, and tolerances that sit
    exactly on elements' |a - r| (atol = d, or rtol = d/|r| in fp64)."""
    torch, kc, ctx, orc = env
    dt = orc.DTYPE_NAMES.index(dtname)
    rng = np.random.default_rng(35 + dt)
    n = 2048
    pairs = []
    for j in range(84):
        r, a = _spread16(dt, n, j % 21, rng, orc, flip=0.0 if j % 3 == 0 else 0.3)
        if j % 7 == 6:   # a few specials on both sides
            rv, av = r.view(np.uint16), a.view(np.uint16)
            ex = 0x7C00 if dt == orc.DT_F16 else 0x7F80
            av[5], rv[9], av[9], rv[13] = ex | 1, ex, ex, ex | 3
        pairs.append((r, a))
    # tolerances on an element's exact |a - r| (fp64, like the oracle)
    f = np.float16 if dt == orc.DT_F16 else None

    def vals(u8):
        u = u8.view(np.uint16)
        if f is not None:
            return u.view(np.float16).astype(np.float64)
        return (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    r0, a0 = vals(pairs[4][0]), vals(pairs[4][1])
    k = int(np.nonzero((r0 != a0) & (r0 != 0) & np.isfinite(r0) & np.isfinite(a0))[0][7])
    d = abs(a0[k] - r0[k])
    tols = [(1e-8, 1e-5, False), (0.0, 0.0, False), (1e-3, 1e-3, True), (d, 0.0, False), (0.0, d / abs(r0[k]), False),
            (1e-2, 0.0, False), (1e-30, 1e-30, False), (float(np.nextafter(d, 0)), 0.0, False)]
    hold, bufs = [], []
    for r, a in pairs:
        tr, pr = _dev(torch, r)
        ta, pa = _dev(torch, a)
        hold += [tr, ta]
        bufs.append((pr, pa, r.size, dtname))
    for tol in tols:
        reps, bms = ctx.diff(bufs, atol=tol[0], rtol=tol[1], equal_nan=tol[2])
        for j, (r, a) in enumerate(pairs):
            exp = orc.diff(r, a, dt, atol=tol[0], rtol=tol[1], equal_nan=tol[2])
            _same(reps[j], exp.report, f"{dtname} buffer {j} tol {tol}")
            assert [int(w) for w in bms[j]] == [int(w) for w in exp.bitmap]


def test_k2_identical_and_empty(env):
    torch, kc, ctx, orc = env
    r, _ = _pair_host(orc.DT_F32, 100000, 1, orc, specials=False)
    tr, pr = _dev(torch, r)
    ta, pa = _dev(torch, r.copy())
    reps, bms = ctx.diff([(pr, pa, r.size, "f32"), (pr, pa, 0, "bytes")])
    assert reps[0]["differing_bytes"] == 0 and reps[0]["pass"] == 1 and reps[0]["max_abs"] == 0.0
    assert reps[1]["nbytes"] == 0 and reps[1]["pass"] == 1
    assert all(w == 0 for w in bms[0])


def test_k2_rejects_partial_elements(env):
    torch, kc, ctx, orc = env
    t = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(kc.KcError):
        ctx.diff([(t.data_ptr(), t.data_ptr(), 6, "f32")])


def test_k2_many_buffers_one_call(env):
    torch, kc, ctx, orc = env
    specs = [("f16", 70000), ("bytes", 130000), ("bf16", 33333 * 2), ("f64", 8 * 9000), ("u16", 2 * 50001)]
    hold, bufs, exps = [], [], []
    for i, (dtn, nb) in enumerate(specs):
        dt = orc.DTYPE_NAMES.index(dtn)
        r, a = _pair_host(dt, nb // orc.ELEM_SIZE[dt], seed=40 + i, orc=orc)
        tr, pr = _dev(torch, r)
        ta, pa = _dev(torch, a)
        hold += [tr, ta]
        bufs.append((pr, pa, r.size, dtn))
        exps.append(orc.diff(r, a, dt))
    reps, bms = ctx.diff(bufs)
    for got, exp, bm in zip(reps, exps, bms):
        _same(got, exp.report)
        assert [int(w) for w in bm] == [int(w) for w in exp.bitmap]


@pytest.mark.parametrize("kind", ["f16", "bf16"])
def test_k2_c3_recipe_moderate(env, kind):
    """c3's planting recipe on a 16 MiB pair, generated on the device."""
    torch, kc, ctx, orc = env
    import synth
    n = 8 * 2**20
    g = torch.Generator(device="cuda").manual_seed(synth.seed(3))
    tdt = torch.float16 if kind == "f16" else torch.bfloat16
    ref = (torch.randn(n, device="cuda", generator=g) * 0.5).to(tdt)
    act = torch.empty_like(ref)
    synth.plant_c3(ref.view(torch.int16), act.view(torch.int16), kind, synth.C3_MISMATCH_P, g)
    torch.cuda.synchronize()
    rh, ah = ref.view(torch.uint8).cpu().numpy(), act.view(torch.uint8).cpu().numpy()
    dt = orc.DT_F16 if kind == "f16" else orc.DT_BF16
    for tol in [(1e-8, 1e-5, False), (1e-3, 1e-3, False), (1e-3, 1e-3, True)]:
        reps, bms = ctx.diff([(ref.data_ptr(), act.data_ptr(), 2 * n, kind)], atol=tol[0], rtol=tol[1],
                             equal_nan=tol[2])
        exp = orc.diff(rh, ah, dt, atol=tol[0], rtol=tol[1], equal_nan=tol[2])
        _same(reps[0], exp.report, f"c3 {kind} {tol}")
        assert [int(w) for w in bms[0]] == [int(w) for w in exp.bitmap]
    # the recipe's closed-form counts: 3+1 NaN in A among finite/differing, 1+2 NaN in R
    assert reps[0]["nan_ref"] == 2 and reps[0]["nan_act"] == 5 and reps[0]["nan_pos_mismatch"] == 3
    assert reps[0]["rel_undefined"] >= 1


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["f16", "bf16"])
def test_k2_c3_full_size(env, kind):
    """Full c3: Q, K, V, O pairs of 536,870,912 B each (4 GiB read), whole-buffer oracle."""
    torch, kc, ctx, orc = env
    import synth
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
    reps, bms = ctx.diff(bufs)
    dt = orc.DT_F16 if kind == "f16" else orc.DT_BF16
    for i, (r, a) in enumerate(zip(refs, acts)):
        exp = orc.diff(r.view(torch.uint8).cpu().numpy(), a.view(torch.uint8).cpu().numpy(), dt)
        _same(reps[i], exp.report, f"c3 full {kind} #{i}")
        assert [int(w) for w in bms[i]] == [int(w) for w in exp.bitmap]
    assert reps[1]["differing_bytes"] == 1 and reps[0]["differing_bytes"] == 0


def test_k2_plan_cache_sees_new_contents_and_new_sets(env):
    """Identical buffer sets reuse the uploaded tables; contents are always re-read."""
    torch, kc, ctx, orc = env
    r, a = _pair_host(orc.DT_F16, 200000, 77, orc)
    tr, pr = _dev(torch, r)
    ta, pa = _dev(torch, a)
    bufs = [(pr, pa, r.size, "f16")]
    first, _ = ctx.diff(bufs)
    _same(first[0], orc.diff(r, a, orc.DT_F16).report, "first")
    a2 = a.copy()
    a2[1000:1100] ^= 0x55
    ta[:a2.size].copy_(torch.from_numpy(a2))
    second, _ = ctx.diff(bufs)                      # same set, new contents
    _same(second[0], orc.diff(r, a2, orc.DT_F16).report, "second")
    third, _ = ctx.diff([(pr, pa, r.size // 2, "f16")])   # a different set
    _same(third[0], orc.diff(r[:r.size // 2], a2[:a2.size // 2], orc.DT_F16).report, "third")


@pytest.mark.parametrize("every,ctas", [("1", ""), ("3", "1"), ("5", "2")])
def test_periodic_flush_path(every, ctas):
    """K2's periodic flush of the 32-bit lane counters (every kFlushUnits = 1 GiB per
    warp in production, which no test-sized launch reaches) forced to every 1 / 3 / 5
    units in a fresh process, with the grid cut to 1 or 2 CTAs so each warp walks
    ~20 units across segment boundaries: reports and bitmaps still equal the oracle's."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "tests", "k2_flush_worker.py")], capture_output=True,
                       text=True, timeout=600, env=dict(os.environ, KC_K2_FLUSH_UNITS=every, KC_K2_MAX_CTAS=ctas))
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["flush_units"] == every and r["bad"] == [], r["bad"][:10]
    assert all(d > 0 for d in r["differing_elems"])


@pytest.mark.parametrize("name", ["f16", "bf16"])
@pytest.mark.parametrize("equal_nan", [False, True])
def test_k2_16bit_every_pattern_against_neighbours(env, name, equal_nan):
    """Every one of the 65,536 16-bit patterns as the reference, against itself, its sign
    flip, its LSB flip, +0, -0, the smallest subnormal and a quiet NaN: the K2 flag scan
    (HSET2-based by default) must send exactly the elements the oracle counts -- equal
    NaNs, +0/-0, subnormal vs zero, Inf vs NaN -- so every report field and bitmap bit
    equals the oracle's."""
    torch, kc, ctx, orc = env
    dt = kc.DT[name]
    pat = np.arange(65536, dtype=np.uint16)
    qnan = np.uint16(0x7E00 if name == "f16" else 0x7FC0)
    partners = [pat, pat ^ np.uint16(0x8000), pat ^ np.uint16(1), np.zeros_like(pat), np.full_like(pat, 0x8000),
                np.full_like(pat, 1), np.full_like(pat, qnan)]
    ref = np.tile(pat, len(partners))
    act = np.concatenate(partners)
    rb, ab = ref.view(np.uint8), act.view(np.uint8)
    dr, pr = _dev(torch, rb)
    da, pa = _dev(torch, ab)
    torch.cuda.synchronize()
    for tol in ((1e-8, 1e-5), (1e-3, 1e-3), (0.0, 0.0)):
        reps, bms = ctx.diff([(pr, pa, rb.size, name)], atol=tol[0], rtol=tol[1], equal_nan=equal_nan)
        exp = orc.diff(rb, ab, dt, atol=tol[0], rtol=tol[1], equal_nan=equal_nan)
        _same(reps[0], exp.report, f"{name} tol={tol} equal_nan={equal_nan}")
        assert [int(x) for x in bms[0]] == [int(x) for x in exp.bitmap]
