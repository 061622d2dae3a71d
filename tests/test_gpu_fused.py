"""GPU parity of F2 (kc_hash_diff_async: K5 fused hash + compare, then K2 over
the dirty chunks only) against the oracle: the manifest of the actual bytes
(O2), each buffer's O4 report and bitmap, bit for bit, and the dirty set is a
valid one (every chunk the oracle's bitmap flags, or whose reference holds an
Inf/NaN, is dirty; every clean chunk is bit-identical)."""
import numpy as np
import pytest

from test_gpu_diff import CH, _dev, _pair_host, _same

pytestmark = pytest.mark.gpu


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


def _special_chunks(r: np.ndarray, dt: int, orc) -> set:
    """Chunks whose reference holds an element with an all-ones exponent."""
    if dt not in (orc.DT_F16, orc.DT_BF16, orc.DT_F32, orc.DT_F64):
        return set()
    ut = {orc.DT_F16: np.uint16, orc.DT_BF16: np.uint16, orc.DT_F32: np.uint32, orc.DT_F64: np.uint64}[dt]
    ex = {orc.DT_F16: 0x7C00, orc.DT_BF16: 0x7F80, orc.DT_F32: 0x7F800000, orc.DT_F64: 0x7FF0000000000000}[dt]
    v = r.view(ut)
    idx = np.nonzero((v & ut(ex)) == ut(ex))[0]
    return set(int(i) * np.dtype(ut).itemsize // CH for i in idx)


def _run(torch, kc, ctx, orc, pairs, tol=(1e-8, 1e-5, False), offsets=None):
    """pairs: [(dtname, ref_u8, act_u8)] -> checks everything against the oracle."""
    keep, bufs = [], []
    for j, (dtname, r, a) in enumerate(pairs):
        off = offsets[j] if offsets else (0, 0)
        tr, pr = _dev(torch, r, off[0])
        ta, pa = _dev(torch, a, off[1])
        keep += [tr, ta]
        bufs.append((pr, pa, r.size, dtname))
    nch = [(r.size + CH - 1) // CH for _, r, _ in pairs]
    C = sum(nch)
    words = [(c + 63) // 64 for c in nch]
    d_h = torch.zeros(max(1, C), dtype=torch.int64, device="cuda")
    d_rep = torch.zeros(max(1, len(pairs)) * 15, dtype=torch.int64, device="cuda")
    d_bm = torch.zeros(max(1, sum(words)), dtype=torch.int64, device="cuda")
    d_dirty = torch.zeros(max(1, (C + 63) // 64), dtype=torch.int64, device="cuda")
    ctx.hash_diff_async(bufs, d_h.data_ptr(), d_rep.data_ptr(), d_bm.data_ptr(), d_dirty.data_ptr(),
                        atol=tol[0], rtol=tol[1], equal_nan=tol[2])
    torch.cuda.synchronize()
    hashes = d_h.cpu().numpy().view(np.uint64)[:C]
    raw = d_rep.cpu().numpy().tobytes()
    bm = d_bm.cpu().numpy().view(np.uint64)
    dirty = d_dirty.cpu().numpy().view(np.uint64)
    c0, w0 = 0, 0
    for j, (dtname, r, a) in enumerate(pairs):
        dt = orc.DTYPE_NAMES.index(dtname)
        exp_h = orc.chunk_hashes(a)
        assert np.array_equal(hashes[c0:c0 + nch[j]], exp_h), f"{dtname} manifest"
        rep = kc.DiffReport.from_buffer_copy(raw[120 * j:120 * (j + 1)]).as_dict()
        exp = orc.diff(r, a, dt, atol=tol[0], rtol=tol[1], equal_nan=tol[2])
        _same(rep, exp.report, f"{dtname} {r.size}")
        assert [int(x) for x in bm[w0:w0 + words[j]]] == [int(x) for x in exp.bitmap], f"{dtname} bitmap"
        # dirty validity
        must = _special_chunks(r, dt, orc)
        for k in range(nch[j]):
            g = c0 + k
            d = (int(dirty[g // 64]) >> (g % 64)) & 1
            lo, hi = k * CH, min(r.size, (k + 1) * CH)
            differs = not np.array_equal(r[lo:hi], a[lo:hi])
            if differs or k in must:
                assert d == 1, f"{dtname} chunk {k} must be dirty"
            if d == 0:
                assert not differs
        c0 += nch[j]
        w0 += words[j]
    return hashes, dirty


ALL_DT = ["bytes", "u8", "i8", "u16", "i16", "u32", "i32", "u64", "i64", "f16", "bf16", "f32", "f64"]


@pytest.mark.parametrize("dtname", ALL_DT)
def test_fused_parity_planted(env, dtname):
    torch, kc, ctx, orc = env
    dt = orc.DTYPE_NAMES.index(dtname)
    s = orc.ELEM_SIZE[dt]
    pairs = []
    for nbytes, dens in [(3 * CH + 40, 0.113), (700 * 1024 + 24, 1e-5), (8, 0.5), (64 * CH, 0.0)]:
        r, a = _pair_host(dt, nbytes // s, seed=nbytes + 7 * dt, orc=orc, specials=dens > 0.1, density=dens)
        pairs.append((dtname, r, a))
    for tol in [(1e-8, 1e-5, False), (1e-3, 1e-3, True)]:
        _run(torch, kc, ctx, orc, pairs, tol)


def test_fused_sparse_dirty_many_buffers(env):
    """Mostly identical buffers with a few planted chunks: the dirty set is
    sparse and clustered, K2 reads only those chunks, results still exact."""
    torch, kc, ctx, orc = env
    rng = np.random.default_rng(11)
    pairs = []
    for j in range(40):
        dtname = ["bf16", "f32", "bytes", "i32"][j % 4]
        n = int(rng.integers(1, 40)) * CH + int(rng.integers(0, 4)) * 32
        r = rng.integers(0, 256, size=n, dtype=np.uint8)
        if dtname == "bf16":  # finite values only
            r = (rng.standard_normal(n // 2).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16).view(np.uint8)
        if dtname == "f32":
            r = rng.standard_normal(n // 4).astype(np.float32).view(np.uint8)
        a = r.copy()
        if j % 3 == 0:
            p = int(rng.integers(0, n // 8)) * 8
            a[p] ^= 0x01
        pairs.append((dtname, r, a))
    hashes, dirty = _run(torch, kc, ctx, orc, pairs)
    total = sum((r.size + CH - 1) // CH for _, r, _ in pairs)
    n_dirty = sum(bin(int(w)).count("1") for w in dirty)
    assert n_dirty < total // 4  # the filter really skips work here


def test_fused_identical_nan_reference_is_dirty(env):
    """Bit-identical buffers whose reference holds NaNs still report them
    (nan_ref, allclose_fail without equal_nan): those chunks must be dirty."""
    torch, kc, ctx, orc = env
    r = np.zeros(5 * CH // 4, dtype=np.float32)
    r[CH // 4 * 3 + 5] = np.nan
    r[CH // 4 * 4 + 9] = np.inf
    u = r.view(np.uint8)
    for tol in [(1e-8, 1e-5, False), (1e-8, 1e-5, True)]:
        hashes, dirty = _run(torch, kc, ctx, orc, [("f32", u, u.copy())], tol)
        assert int(dirty[0]) == 0b11000


def test_fused_unaligned_falls_back(env):
    torch, kc, ctx, orc = env
    r, a = _pair_host(orc.DT_F16, (2 * CH + 100) // 2, seed=3, orc=orc)
    _run(torch, kc, ctx, orc, [("f16", r, a)], offsets=[(2, 6)])


def test_fused_matches_k1_and_k2(env):
    """Same buffers through kc_hash + kc_diff and through the fused call."""
    torch, kc, ctx, orc = env
    r, a = _pair_host(orc.DT_BF16, 9 * CH // 2 + 16, seed=4, orc=orc, density=0.001)
    tr, pr = _dev(torch, r)
    ta, pa = _dev(torch, a)
    reps, bms = ctx.diff([(pr, pa, r.size, "bf16")])
    C = (a.size + CH - 1) // CH
    d_h1 = torch.zeros(C, dtype=torch.int64, device="cuda")
    ctx.hash([(pa, a.size)], d_h1.data_ptr())
    torch.cuda.synchronize()
    hashes, _ = _run(torch, kc, ctx, orc, [("bf16", r, a)])
    assert [int(x) for x in d_h1.cpu().numpy().view(np.uint64)] == [int(x) for x in hashes]
    assert reps[0]["differing_elems"] > 0
