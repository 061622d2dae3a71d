"""Prepared plans (kc_hash_plan_* / kc_diff_plan_*): the same region / buffer set
validated and uploaded once, then run many times.  Every run must equal the
per-call kc_hash / kc_diff_async bit for bit, and the oracle (O2 / O4)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
CH = 65536


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


def _regions(torch, rng, sizes, align=256):
    offs = np.concatenate([[0], np.cumsum((np.asarray(sizes) + align - 1) // align * align)])
    buf = torch.randint(0, 256, (int(offs[-1]) + 64,), dtype=torch.uint8, device="cuda")
    return buf, [(buf.data_ptr() + int(o), int(s)) for o, s in zip(offs[:-1], sizes)]


@pytest.mark.parametrize("kind", ["ragged", "many_small", "unaligned"])
def test_hash_plan_equals_kc_hash_and_oracle(env, kind):
    torch, kc, ctx, orc = env
    rng = np.random.default_rng({"ragged": 1, "many_small": 2, "unaligned": 3}[kind])
    if kind == "ragged":
        sizes = [CH * 5 + 17, 1, CH, 3 * CH - 1, 40000, CH * 9]
        align = 256
    elif kind == "many_small":
        sizes = list(4096 + rng.integers(0, 4096, size=3000))
        align = 256
    else:
        sizes = [CH + 3, 1000, 2 * CH + 5]
        align = 8          # bases not 16-byte aligned: the generic K1
    buf, regions = _regions(torch, rng, sizes, align)
    if kind == "unaligned":
        regions = [(b + 3, s) for b, s in regions]
    C = kc.count_chunks(regions)
    n = len(regions)
    plan = ctx.hash_plan(regions)
    assert plan.chunks == C
    a = torch.zeros(C, dtype=torch.int64, device="cuda")
    b = torch.zeros(C, dtype=torch.int64, device="cuda")
    da = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    db = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    for _ in range(3):
        plan.run(a.data_ptr(), da.data_ptr(), da.data_ptr() + 8 * n)
    ctx.hash(regions, b.data_ptr(), db.data_ptr(), db.data_ptr() + 8 * n)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(da, db)
    host = buf.cpu().numpy()
    base0 = buf.data_ptr()
    exp = np.concatenate([orc.chunk_hashes(host[bb - base0:bb - base0 + s]) for bb, s in regions])
    assert np.array_equal(a.cpu().numpy().view(np.uint64), exp)
    plan.close()


def test_diff_plan_equals_kc_diff_async_and_oracle(env):
    torch, kc, ctx, orc = env
    rng = np.random.default_rng(7)
    names = ["bf16", "f16", "f32", "bytes", "i32", "u64"]
    bufs, host = [], []
    keep = []
    for i, nm in enumerate(names):
        es = orc.ELEM_SIZE[kc.DT[nm]]
        nb = (3 * CH + 4096 * i + 8) // es * es
        r = rng.integers(0, 256, nb, dtype=np.uint8)
        if nm in ("bf16", "f16", "f32"):
            r = (rng.standard_normal(nb // es).astype(np.float32)).view(np.uint8) if nm == "f32" else \
                (rng.standard_normal(nb // 2).astype(np.float16).view(np.uint8) if nm == "f16" else
                 (rng.standard_normal(nb // 2).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16).view(np.uint8))
        a = r.copy()
        for o in rng.integers(0, nb, size=40):
            a[o] ^= 1 << int(rng.integers(0, 8))
        dr = torch.from_numpy(r).cuda()
        da = torch.from_numpy(a).cuda()
        keep += [dr, da]
        bufs.append((dr.data_ptr(), da.data_ptr(), nb, nm))
        host.append((r, a, kc.DT[nm]))
    nbytes = [b[2] for b in bufs]
    word0, acc = [], 0
    for n in nbytes:
        word0.append(acc)
        acc += ((n + CH - 1) // CH + 63) // 64
    plan = ctx.diff_plan(bufs, len(bufs), nbytes, word0)
    r1 = torch.zeros(len(bufs) * 15, dtype=torch.int64, device="cuda")
    r2 = torch.zeros_like(r1)
    b1 = torch.zeros(acc, dtype=torch.int64, device="cuda")
    b2 = torch.zeros_like(b1)
    for tol in ((1e-8, 1e-5), (1e-3, 1e-3)):
        plan.run(r1.data_ptr(), b1.data_ptr(), atol=tol[0], rtol=tol[1])
        plan.run(r1.data_ptr(), b1.data_ptr(), atol=tol[0], rtol=tol[1])   # reruns re-zero the reports
        ctx.diff_async(bufs, len(bufs), nbytes, r2.data_ptr(), word0, b2.data_ptr(), atol=tol[0], rtol=tol[1])
        torch.cuda.synchronize()
        assert torch.equal(r1, r2) and torch.equal(b1, b2)
        raw = r1.cpu().numpy().tobytes()
        bm = b1.cpu().numpy().view(np.uint64)
        for j, (r, a, dt) in enumerate(host):
            got = kc.DiffReport.from_buffer_copy(raw[120 * j:120 * (j + 1)]).as_dict()
            exp = orc.diff(r, a, dt, atol=tol[0], rtol=tol[1])
            for f, v in exp.report.items():
                assert got[f] == v or (isinstance(v, float) and np.isnan(got[f]) and np.isnan(v)), (names[j], f)
            nw = ((r.size + CH - 1) // CH + 63) // 64
            assert [int(x) for x in bm[word0[j]:word0[j] + nw]] == [int(x) for x in exp.bitmap]
    plan.close()


def test_plan_errors(env):
    torch, kc, ctx, orc = env
    buf = torch.zeros(4 * CH, dtype=torch.uint8, device="cuda")
    b = buf.data_ptr()
    # an unsorted set cannot give the snapshot digest (R25); the manifest is fine
    plan = ctx.hash_plan([(b + 2 * CH, CH), (b, CH)])
    out = torch.zeros(3, dtype=torch.int64, device="cuda")
    plan.run(out.data_ptr())
    with pytest.raises(kc.KcError):
        plan.run(out.data_ptr(), 0, out.data_ptr() + 16)
    plan.close()
    with pytest.raises(kc.KcError):
        ctx.hash_plan([(b, 0)])
    # a plan made without bitmap offsets takes no bitmaps; a plan of another context is refused
    dp = ctx.diff_plan([(b, b + CH, CH, "bytes")], 1, [CH])
    reps = torch.zeros(15, dtype=torch.int64, device="cuda")
    dp.run(reps.data_ptr())
    with pytest.raises(kc.KcError):
        dp.run(reps.data_ptr(), out.data_ptr())
    other = kc.Context(0)
    with pytest.raises(kc.KcError):
        kc.DiffPlan(other, dp._h).run(reps.data_ptr())
    other.close()
    dp.close()
    with pytest.raises(kc.KcError):
        ctx.diff_plan([(b, b + CH, CH, "f32", 3)], 1, [CH])     # report index out of range
