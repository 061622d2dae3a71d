"""Pins for the oracle's O4 diff report.

Pins: brute-force numpy byte compare (counts, bitmap); SPEC.md:673's printed
percent example; IEEE closed-form ULP cases (golden); an exhaustive
sorted-rank definition of ULP distance for f16/bf16 ("how many representable
values apart"); np.nextafter stepping for f32/f64; numpy float64 for max
abs/rel; np.isclose for the allclose count; np.isnan for NaN counters; Python
integers for integer distances; hypothesis properties.
"""
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _bits_to_f64(bits, dt, orc):
    """Exact fp64 values of raw element bits via numpy's own conversions."""
    if dt == orc.DT_F16:
        return bits.astype(np.uint16).view(np.float16).astype(np.float64)
    if dt == orc.DT_BF16:
        return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if dt == orc.DT_F32:
        return bits.astype(np.uint32).view(np.float32).astype(np.float64)
    return bits.astype(np.uint64).view(np.float64)


NP_UINT = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}


# ----------------------------------------------------------------- bytes, bitmap
@pytest.mark.parametrize("n", [1, 7, 4096, 65536, 65537, 131072 + 3, 300000])
def test_byte_counts_and_bitmap_brute_force(orc, n):
    rng = np.random.default_rng(n)
    r = rng.integers(0, 256, size=n, dtype=np.uint8)
    a = r.copy()
    offs = {0, n - 1, min(n - 1, 65535), min(n - 1, 65536)} | set(int(x) for x in rng.integers(0, n, size=5))
    for o in offs:
        a[o] = (int(a[o]) + 1 + int(rng.integers(0, 254))) % 256
    res = orc.diff(r, a, orc.DT_BYTES)
    rep = res.report
    diffmask = r != a
    assert rep["differing_bytes"] == int(diffmask.sum())
    assert rep["differing_elems"] == int(diffmask.sum())
    assert rep["max_ulp"] == int(np.abs(a.astype(np.int64) - r.astype(np.int64)).max())
    assert rep["percent_bytes"] == 100.0 * diffmask.sum() / n
    nck = (n + 65535) // 65536
    expect = np.zeros((nck + 63) // 64, dtype=np.uint64)
    for k in range(nck):
        if diffmask[k * 65536:(k + 1) * 65536].any():
            expect[k // 64] |= np.uint64(1) << np.uint64(k % 64)
    assert np.array_equal(res.bitmap, expect)
    assert rep["pass"] == 0
    assert orc.diff(r, r, orc.DT_BYTES).report["pass"] == 1


def test_percent_printed_example(orc):
    vals = {}
    with open(os.path.join(GOLDEN, "percent_example.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()
                vals[k] = v
    n = int(vals["nbytes"])
    r = np.zeros(n, dtype=np.uint8)
    a = r.copy()
    a[int(vals["flipped_offset"])] = 1
    rep = orc.diff(r, a).report
    assert rep["differing_bytes"] == int(vals["differing_bytes"])
    assert rep["percent_bytes"] == float(vals["percent_bytes"])


def test_bitmap_many_chunks(orc):
    n = 130 * 65536 + 5
    r = np.zeros(n, dtype=np.uint8)
    a = r.copy()
    chunks = [0, 63, 64, 65, 127, 128, 130]
    for k in chunks:
        a[min(n - 1, k * 65536 + 100)] = 9
    bm = orc.diff(r, a).bitmap
    got = [k for k in range(131) if (int(bm[k // 64]) >> (k % 64)) & 1]
    assert got == chunks


def test_size_not_multiple_of_element_rejected(orc):
    with pytest.raises(ValueError):
        orc.diff(np.zeros(5, np.uint8), np.zeros(5, np.uint8), orc.DT_F32)


# ----------------------------------------------------------------- ULP
def _golden_ulp():
    out = []
    with open(os.path.join(GOLDEN, "ulp_special_cases.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                p = line.split()
                out.append((p[0], int(p[1], 16), int(p[2], 16), int(p[3], 16) if p[0] == "f64" else int(p[3])))
    return out


@pytest.mark.parametrize("dtname,rbits,abits,expect", _golden_ulp())
def test_ulp_special_cases(orc, dtname, rbits, abits, expect):
    dt = {"f16": orc.DT_F16, "bf16": orc.DT_BF16, "f32": orc.DT_F32, "f64": orc.DT_F64}[dtname]
    s = orc.ELEM_SIZE[dt]
    r = np.array([rbits], dtype=NP_UINT[s])
    a = np.array([abits], dtype=NP_UINT[s])
    assert orc.diff(r, a, dt).report["max_ulp"] == expect


def _rank_table(dt, orc):
    """Independent ULP definition: rank of each non-NaN pattern among all
    distinct representable values (+0 and -0 are one value)."""
    bits = np.arange(65536, dtype=np.uint64)
    vals = _bits_to_f64(bits, dt, orc)
    ok = ~np.isnan(vals)
    uniq = np.unique(vals[ok])
    rank = np.full(65536, -1, dtype=np.int64)
    rank[ok] = np.searchsorted(uniq, vals[ok])
    return rank


@pytest.mark.parametrize("dtname", ["f16", "bf16"])
def test_ulp_exhaustive_rank_definition(orc, dtname):
    dt = orc.DT_F16 if dtname == "f16" else orc.DT_BF16
    rank = _rank_table(dt, orc)
    valid = np.nonzero(rank >= 0)[0]
    rng = np.random.default_rng(5)
    # random far pairs, near pairs, and pairs straddling zero
    pairs = list(zip(rng.choice(valid, 400), rng.choice(valid, 400)))
    for b in rng.choice(valid, 200):
        for k in (1, 2, 3, 16):
            pairs.append((b, b + k if b + k < 65536 and rank[(b + k)] >= 0 else b))
    pairs += [(0x0000, 0x8000), (0x0001, 0x8001), (0x8001, 0x0002), (0x8000, 0x0003)]
    # one element per pair would be many ctypes calls; pack each pair as a
    # 1-element buffer and check max_ulp for each
    for rb, ab in pairs:
        r = np.array([rb], dtype=np.uint16)
        a = np.array([ab], dtype=np.uint16)
        got = orc.diff(r, a, dt).report["max_ulp"]
        assert got == abs(int(rank[ab]) - int(rank[rb])), (hex(rb), hex(ab))


@pytest.mark.parametrize("dtname", ["f32", "f64"])
def test_ulp_nextafter_stepping(orc, dtname):
    npt = np.float32 if dtname == "f32" else np.float64
    dt = orc.DT_F32 if dtname == "f32" else orc.DT_F64
    ut = np.uint32 if dtname == "f32" else np.uint64
    rng = np.random.default_rng(9)
    starts = list(rng.standard_normal(40).astype(npt)) + [npt(0.0), npt(-0.0), npt(np.finfo(npt).tiny),
                                                           npt(-np.finfo(npt).smallest_subnormal),
                                                           npt(np.finfo(npt).max)]
    for x in starts:
        for k in (1, 2, 5, 17):
            toward = npt(-np.inf) if rng.random() < 0.5 else npt(np.inf)
            y = x
            steps = 0
            while steps < k and not np.isinf(y):
                y = np.nextafter(y, toward)
                # +0 and -0 are one point: nextafter(-0, +) jumps to +min subnormal
                steps += 1
            r = np.array([x], dtype=npt).view(ut)
            a = np.array([y], dtype=npt).view(ut)
            got = orc.diff(r, a, dt).report["max_ulp"]
            # a bit-level 0 vs -0 pair is distance 0; numpy may emit -0 on the way
            expect = steps
            if x == 0 and y == 0:
                expect = 0
            assert got == expect, (x, y, k)


# ----------------------------------------------------------------- abs / rel / allclose / NaN
def _float_case(dt, orc, n, seed, specials=True):
    rng = np.random.default_rng(seed)
    s = orc.ELEM_SIZE[dt]
    if dt == orc.DT_F16:
        r = rng.standard_normal(n).astype(np.float16).view(np.uint16)
    elif dt == orc.DT_BF16:
        r = (rng.standard_normal(n).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    elif dt == orc.DT_F32:
        r = rng.standard_normal(n).astype(np.float32).view(np.uint32)
    else:
        r = rng.standard_normal(n).view(np.uint64)
    r = r.copy()
    a = r.copy()
    ut = NP_UINT[s]
    # +-k ULP shifts on a Bernoulli(0.113) subset (the paper's 11.3%)
    m = rng.random(n) < 0.113
    k = np.where(rng.random(n) < 0.9, 1, rng.integers(2, 17, size=n)).astype(np.int64)
    sign = np.where(rng.random(n) < 0.5, -1, 1)
    a[m] = (a[m].astype(np.int64) + (sign * k)[m]).astype(ut)
    if specials and n >= 16:
        sign_bit = 1 << (8 * s - 1)
        exp_all = {orc.DT_F16: 0x7C00, orc.DT_BF16: 0x7F80, orc.DT_F32: 0x7F800000,
                   orc.DT_F64: 0x7FF0000000000000}[dt]
        qnan = exp_all | (exp_all >> 1 & ~exp_all) | 1
        a[1] = qnan                       # A NaN, R finite
        r[2] = qnan; a[2] = qnan          # both NaN, same payload
        r[3] = qnan; a[3] = qnan | 2      # both NaN, different payload
        a[4] = exp_all                    # A = +inf
        r[5] = 0; a[5] = sign_bit         # +0 vs -0
        r[6] = 0; a[6] = 1                # 0 vs min subnormal -> rel undefined
        a[7] = r[7] ^ sign_bit            # A = -R
        r[8] = exp_all; a[8] = exp_all    # both +inf (bit-equal)
        r[9] = exp_all; a[9] = exp_all | sign_bit  # +inf vs -inf
        r[10] = exp_all                   # R = +inf, A finite
    return r, a


def _numpy_expect(r, a, dt, orc, atol, rtol, equal_nan):
    r64 = _bits_to_f64(r, dt, orc)
    a64 = _bits_to_f64(a, dt, orc)
    nr, na = np.isnan(r64), np.isnan(a64)
    differ = r != a
    mask = differ & ~nr & ~na
    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        d = np.abs(a64 - r64)
        max_abs = float(d[mask].max()) if mask.any() else 0.0
        relmask = mask & (d != 0)
        undef = relmask & (r64 == 0)
        rr = relmask & ~undef
        rel = np.where(np.isinf(r64[rr]), np.inf, d[rr] / np.abs(r64[rr]))
        max_rel = float(rel.max()) if rel.size else 0.0
        close = np.isclose(a64, r64, rtol=rtol, atol=atol, equal_nan=equal_nan)
    return dict(differing_elems=int(differ.sum()), max_abs=max_abs, max_rel=max_rel,
                rel_undefined=int(undef.sum()), nan_ref=int(nr.sum()), nan_act=int(na.sum()),
                nan_pos_mismatch=int((nr ^ na).sum()), allclose_fail=int((~close).sum()))


@pytest.mark.parametrize("dtname", ["f16", "bf16", "f32", "f64"])
@pytest.mark.parametrize("tol", [(1e-8, 1e-5, False), (1e-3, 1e-3, False), (1e-3, 1e-3, True), (0.0, 0.0, True)])
def test_float_report_vs_numpy(orc, dtname, tol):
    dt = {"f16": orc.DT_F16, "bf16": orc.DT_BF16, "f32": orc.DT_F32, "f64": orc.DT_F64}[dtname]
    atol, rtol, eqn = tol
    r, a = _float_case(dt, orc, 5000, seed=dt)
    rep = orc.diff(r, a, dt, atol=atol, rtol=rtol, equal_nan=eqn).report
    exp = _numpy_expect(r, a, dt, orc, atol, rtol, eqn)
    for key, v in exp.items():
        assert rep[key] == v, (key, rep[key], v)
    assert rep["pass"] == int(exp["allclose_fail"] == 0)


def test_bit_equal_nan_fails_strict_passes_equal_nan(orc):
    # PAPER.md:1132-1135 (NaNs reported explicitly); reading R15
    r = np.array([0x7E00, 0x3C00], dtype=np.uint16)
    rep0 = orc.diff(r, r.copy(), orc.DT_F16, equal_nan=False).report
    rep1 = orc.diff(r, r.copy(), orc.DT_F16, equal_nan=True).report
    assert rep0["allclose_fail"] == 1 and rep0["pass"] == 0 and rep0["nan_ref"] == 1 and rep0["differing_elems"] == 0
    assert rep1["allclose_fail"] == 0 and rep1["pass"] == 1


# ----------------------------------------------------------------- integers
@pytest.mark.parametrize("dtname,npt", [("u8", np.uint8), ("i8", np.int8), ("u16", np.uint16), ("i16", np.int16),
                                         ("u32", np.uint32), ("i32", np.int32), ("u64", np.uint64),
                                         ("i64", np.int64)])
def test_integer_distance_python_ints(orc, dtname, npt):
    dt = orc.DTYPE_NAMES.index(dtname)
    info = np.iinfo(npt)
    rng = np.random.default_rng(dt)
    r = rng.integers(info.min, info.max, size=300, dtype=npt, endpoint=True)
    a = r.copy()
    a[:100] = rng.integers(info.min, info.max, size=100, dtype=npt, endpoint=True)
    a[100] = info.max
    r[100] = info.min
    rep = orc.diff(r, a, dt).report
    expect = max(abs(int(x) - int(y)) for x, y in zip(a.tolist(), r.tolist()))
    assert rep["max_ulp"] == expect
    assert rep["differing_elems"] == int((r != a).sum())
    assert rep["pass"] == 0
    assert rep["max_abs"] == 0.0 and rep["allclose_fail"] == 0


# ----------------------------------------------------------------- properties
@settings(max_examples=60, deadline=None)
@given(st.binary(min_size=0, max_size=600), st.binary(min_size=0, max_size=600))
def test_symmetry_differing_bytes(orc, x, y):
    n = min(len(x), len(y))
    a = orc.diff(x[:n], y[:n]).report
    b = orc.diff(y[:n], x[:n]).report
    assert a["differing_bytes"] == b["differing_bytes"]
    assert a["max_ulp"] == b["max_ulp"]


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 2**32 - 1), st.floats(0, 1e-2), st.floats(0, 1e-2), st.floats(0, 1e-1), st.floats(0, 1e-1))
def test_tolerance_monotonicity(orc, seed, atol, rtol, datol, drtol):
    r, a = _float_case(orc.DT_F32, orc, 256, seed=seed, specials=False)
    f1 = orc.diff(r, a, orc.DT_F32, atol=atol, rtol=rtol).report["allclose_fail"]
    f2 = orc.diff(r, a, orc.DT_F32, atol=atol + datol, rtol=rtol + drtol).report["allclose_fail"]
    assert f2 <= f1
