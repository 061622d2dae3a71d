"""F2 hash-filtered validation against a host-resident reference
(kc_validate_host_ref; R34) vs the oracle's O4.

The reference lives in host memory with its manifest (computed by the
oracle); the actual buffers live on the device.  Planted cases per dtype:
mismatching chunks (only those cross PCIe), a NaN pair and an Inf pair in
chunks whose bytes are equal (their hashes match: compared with themselves,
they still count NaNs and fail strict allclose), a stale manifest entry (hash
says dirty, bytes equal), ragged tails.  Every report field and bitmap must
equal oracle.diff(ref, act) exactly, and h2d bytes must be the manifest plus
exactly the dirty chunks.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CH = 65536
FIELDS = ["nbytes", "n_elems", "n_chunks", "differing_bytes", "differing_elems", "max_ulp", "max_abs", "max_rel",
          "percent_bytes", "nan_ref", "nan_act", "nan_pos_mismatch", "rel_undefined", "allclose_fail", "pass"]


@pytest.fixture(scope="module")
def env():
    import torch

    import oracle
    from paper_2605_03208_b200 import build, kc
    build.build()
    oracle.build()
    torch.cuda.set_device(0)
    ctx = kc.Context(0)
    yield torch, kc, ctx, oracle
    ctx.close()


def _case(orc, dt, n_chunks, tail, seed, dirty_chunks, nan_chunk, inf_chunk):
    rng = np.random.default_rng(seed)
    es = orc.ELEM_SIZE[dt]
    nbytes = n_chunks * CH + tail
    nbytes -= nbytes % es
    if dt == orc.DT_BF16:
        ref = (rng.standard_normal(nbytes // 2).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    elif dt == orc.DT_F16:
        ref = rng.standard_normal(nbytes // 2).astype(np.float16).view(np.uint16)
    elif dt == orc.DT_F32:
        ref = rng.standard_normal(nbytes // 4).astype(np.float32).view(np.uint32)
    else:
        ref = rng.integers(0, 256, nbytes, dtype=np.uint8)
    ref = ref.view(np.uint8).copy()
    act = ref.copy()
    for c in dirty_chunks:           # a few +-1 element shifts inside the chunk (ULP-level for floats)
        lo = c * CH
        hi = min(nbytes, lo + CH)
        idx = lo + es * rng.choice((hi - lo) // es, size=min(37, (hi - lo) // es), replace=False)
        for i in idx:
            act[i] ^= 1
    if dt in orc.FLOAT_DTYPES:
        nan = {orc.DT_BF16: (0x7FC1).to_bytes(2, "little"), orc.DT_F16: (0x7E01).to_bytes(2, "little"),
               orc.DT_F32: (0x7FC00001).to_bytes(4, "little")}[dt]
        inf = {orc.DT_BF16: (0x7F80).to_bytes(2, "little"), orc.DT_F16: (0x7C00).to_bytes(2, "little"),
               orc.DT_F32: (0x7F800000).to_bytes(4, "little")}[dt]
        for c, pat in ((nan_chunk, nan), (inf_chunk, inf)):
            if c is not None:
                o = c * CH + 10 * es
                ref[o:o + es] = np.frombuffer(pat, dtype=np.uint8)
                act[o:o + es] = np.frombuffer(pat, dtype=np.uint8)
    return ref, act


CASES = [
    ("bf16", 6, 130, [1, 4], 2, 3),
    ("f16", 5, 66, [0], None, 4),
    ("f32", 4, 4 * 1000 + 12, [3], 1, None),
    ("bytes", 3, 17, [2], None, None),
]


@pytest.mark.parametrize("stale", [False, True])
def test_host_ref_matches_oracle(env, stale):
    torch, kc, ctx, orc = env
    dts = {"bf16": orc.DT_BF16, "f16": orc.DT_F16, "f32": orc.DT_F32, "bytes": orc.DT_BYTES}
    refs, acts, mans, bufs, dirty_bytes = [], [], [], [], 0
    for k, (name, nch, tail, dirty, nanc, infc) in enumerate(CASES):
        dt = dts[name]
        ref, act = _case(orc, dt, nch, tail, 260503208 + 31 * k, dirty, nanc, infc)
        h_ref = torch.from_numpy(ref).pin_memory()
        d_act = torch.from_numpy(act).cuda()
        man = orc.chunk_hashes(ref).copy()
        if stale and k == 0:
            man[5] ^= 0xDEADBEEF      # stale entry: hash says dirty, bytes are equal
        refs.append(h_ref)
        acts.append(d_act)
        mans.append(man)
        bufs.append((h_ref.data_ptr(), d_act.data_ptr(), ref.size, name))
        hd = {c for c in range(orc.n_chunks(ref.size))
              if not np.array_equal(ref[c * CH:(c + 1) * CH], act[c * CH:(c + 1) * CH]) or man[c] != orc.chunk_hashes(ref)[c]}
        dirty_bytes += sum(min(CH, ref.size - c * CH) for c in hd)
    allman = np.ascontiguousarray(np.concatenate(mans))
    torch.cuda.synchronize()
    reps, bms, moved = ctx.validate_host_ref(bufs, allman.ctypes.data)
    for k, (name, *_r) in enumerate(CASES):
        exp = orc.diff(refs[k].numpy(), acts[k].cpu().numpy(), dts[name])
        for f in FIELDS:
            g, e = reps[k][f], exp.report[f]
            assert g == e or (isinstance(e, float) and np.isnan(g) and np.isnan(e)), f"{name} {f}: {g} vs {e}"
        assert [int(x) for x in bms[k]] == [int(x) for x in exp.bitmap], name
    assert moved == allman.nbytes + dirty_bytes
    # the NaN pairs sit in chunks with equal bytes: they are counted anyway
    assert reps[0]["nan_ref"] == 1 and reps[0]["allclose_fail"] >= 1


def test_host_ref_clean_copy_moves_only_the_manifest(env):
    torch, kc, ctx, orc = env
    rng = np.random.default_rng(7)
    ref = rng.integers(0, 256, 9 * CH + 100, dtype=np.uint8)
    h = torch.from_numpy(ref).pin_memory()
    d = torch.from_numpy(ref).cuda()
    man = np.ascontiguousarray(orc.chunk_hashes(ref))
    reps, _, moved = ctx.validate_host_ref([(h.data_ptr(), d.data_ptr(), ref.size, "bytes")], man.ctypes.data)
    assert moved == man.nbytes and reps[0]["differing_bytes"] == 0 and reps[0]["pass"] == 1


def test_host_ref_byte_exact_mode_streams_every_byte(env):
    """ref_manifest == NULL: every reference byte crosses PCIe through the 3 x 256 MiB
    staging ring (a 1 GiB + 2 MiB buffer wraps the ring: 5 pieces), mixed with the small
    CASES packed into shared pieces.  Reports, bitmaps and the act manifest equal the
    oracle's O4 / O2 over the full buffers; h2d bytes = every reference byte."""
    torch, kc, ctx, orc = env
    dts = {"bf16": orc.DT_BF16, "f16": orc.DT_F16, "f32": orc.DT_F32, "bytes": orc.DT_BYTES}
    refs, acts, bufs, names = [], [], [], []
    for k, (name, nch, tail, dirty, nanc, infc) in enumerate(CASES):
        ref, act = _case(orc, dts[name], nch, tail, 260503208 + 77 * k, dirty, nanc, infc)
        refs.append(ref)
        acts.append(act)
        names.append(name)
    # the big one: bf16 N(0,1) with +-1 ULP plants at piece boundaries, a NaN and a ragged tail
    rng = np.random.default_rng(260503208 + 99)
    nb = (1 << 30) + (2 << 20) + 6
    big = (rng.standard_normal(nb // 2).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    bact = big.copy()
    P = (256 << 20) // 2
    for e in (0, P - 1, P, 2 * P + 5, 3 * P - 1, 4 * P + 3, nb // 2 - 1):
        bact[e] ^= 1
    bact[3 * P + 11] = 0x7FC1
    refs.insert(2, big.view(np.uint8))
    acts.insert(2, bact.view(np.uint8))
    names.insert(2, "bf16")
    h_refs = [torch.from_numpy(r).pin_memory() for r in refs]
    d_acts = [torch.from_numpy(a).cuda() for a in acts]
    bufs = [(h.data_ptr(), d.data_ptr(), r.size, nm) for h, d, r, nm in zip(h_refs, d_acts, refs, names)]
    C = sum(orc.n_chunks(r.size) for r in refs)
    d_man = torch.zeros(C, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):   # a second call reuses the ring (the copy stream waits for the previous K2)
        reps, bms, moved = ctx.validate_host_ref(bufs, 0, d_act_manifest=d_man.data_ptr())
        assert moved == sum(r.size for r in refs)
        for k, nm in enumerate(names):
            exp = orc.diff(refs[k], acts[k], dts[nm])
            for f in FIELDS:
                g, e = reps[k][f], exp.report[f]
                assert g == e or (isinstance(e, float) and np.isnan(g) and np.isnan(e)), f"{k} {nm} {f}: {g} vs {e}"
            assert [int(x) for x in bms[k]] == [int(x) for x in exp.bitmap], f"{k} {nm} bitmap"
    want = np.concatenate([orc.chunk_hashes(a, threads=8) for a in acts])
    assert np.array_equal(d_man.cpu().numpy().view(np.uint64), want)
    assert reps[2]["differing_elems"] == 8 and reps[2]["nan_act"] == 1


def test_host_ref_byte_exact_packing_and_edges(env):
    """Byte-exact mode: many small buffers packed into shared staging pieces, one buffer
    exactly one piece long (256 MiB) right after them (so it starts mid-piece and is cut),
    a 1-byte buffer, an empty call.  Every report and bitmap equals the oracle's."""
    torch, kc, ctx, orc = env
    reps, bms, moved = ctx.validate_host_ref([], 0)
    assert reps == [] and moved == 0
    rng = np.random.default_rng(11)
    sizes = [int(x) for x in rng.integers(1, 3 * CH, size=300)] + [256 << 20, 1, 5 * CH + 3]
    refs, acts, bufs, keep = [], [], [], []
    for i, n in enumerate(sizes):
        r = rng.integers(0, 256, n, dtype=np.uint8)
        a = r.copy()
        if i % 3 == 0:
            a[rng.integers(0, n)] ^= 0x40
        if n == 256 << 20:
            a[[0, CH - 1, (128 << 20) + 5, n - 1]] ^= 1
        h = torch.from_numpy(r).pin_memory()
        d = torch.from_numpy(a).cuda()
        keep += [h, d]
        refs.append(r)
        acts.append(a)
        bufs.append((h.data_ptr(), d.data_ptr(), n, "bytes"))
    torch.cuda.synchronize()
    reps, bms, moved = ctx.validate_host_ref(bufs, 0)
    assert moved == sum(sizes)
    for k, (r, a) in enumerate(zip(refs, acts)):
        exp = orc.diff(r, a, orc.DT_BYTES)
        for f in FIELDS:
            assert reps[k][f] == exp.report[f], (k, sizes[k], f, reps[k][f], exp.report[f])
        assert [int(x) for x in bms[k]] == [int(x) for x in exp.bitmap], (k, sizes[k])
