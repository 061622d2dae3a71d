"""GPU parity of K1 (chunk hash + digests) and K3 (written set) against the oracle.

Bit-exact: every chunk hash, region digest, snapshot digest and W word must
equal the oracle's on the same bytes (north star: "bit-exact against the
oracle for hashes, bitmaps")."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CH = 65536


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


def _rand_dev(torch, n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)


def _hash(torch, ctx, regions, digests=True):
    from paper_2605_03208_b200 import kc
    C = kc.count_chunks(regions)
    h = torch.zeros(max(1, C), dtype=torch.int64, device="cuda")
    d = torch.zeros(max(1, len(regions)), dtype=torch.int64, device="cuda")
    s = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.hash(regions, h.data_ptr(), d.data_ptr() if digests else 0, s.data_ptr() if digests else 0,
             stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    u = lambda t: t.cpu().numpy().view(np.uint64)
    return u(h)[:C], u(d)[:len(regions)], int(u(s)[0])


SIZES = [1, 7, 31, 32, 33, 63, 64, 100, 4095, 65535, 65536, 65537, 3 * CH, 3 * CH + 17, 5 * 2**20 + 1001]


def test_k1_bit_exact_edge_lengths(env):
    torch, kc, ctx, orc = env
    bufs = [_rand_dev(torch, n, 100 + i) for i, n in enumerate(SIZES)]
    order = sorted(range(len(bufs)), key=lambda i: bufs[i].data_ptr())
    regions = [(bufs[i].data_ptr(), bufs[i].numel()) for i in order]
    h, d, s = _hash(torch, ctx, regions)
    off = 0
    dig = []
    for (base, size), i in zip(regions, order):
        host = bufs[i].cpu().numpy()
        exp = orc.chunk_hashes(host)
        assert np.array_equal(h[off:off + exp.size], exp), f"size {size}"
        dig.append(orc.region_digest(exp))
        assert int(d[len(dig) - 1]) == dig[-1]
        off += exp.size
    assert off == h.size
    assert s == orc.snapshot_digest([r[0] for r in regions], [r[1] for r in regions], dig)


@pytest.mark.parametrize("misalign", [1, 3, 8, 13])
def test_k1_unaligned_bases_generic_path(env, misalign):
    torch, kc, ctx, orc = env
    big = _rand_dev(torch, 3 * CH + 4096, 7 + misalign)
    regions = [(big.data_ptr() + misalign, 2 * CH + 77), (big.data_ptr() + misalign + 2 * CH + 200, 33)]
    h, _, _ = _hash(torch, ctx, regions, digests=False)
    host = big.cpu().numpy()
    exp = np.concatenate([orc.chunk_hashes(host[misalign:misalign + 2 * CH + 77]),
                          orc.chunk_hashes(host[misalign + 2 * CH + 200:misalign + 2 * CH + 233])])
    assert np.array_equal(h, exp)


def test_k1_many_small_regions(env):
    torch, kc, ctx, orc = env
    # 3000 regions of 4 KiB + jitter carved from one buffer (16-byte aligned bases)
    rng = np.random.default_rng(3)
    sizes = 4096 + rng.integers(0, 4096, size=3000)
    offs = np.concatenate([[0], np.cumsum((sizes + 15) // 16 * 16 + 16)])
    big = _rand_dev(torch, int(offs[-1]), 5)
    regions = [(big.data_ptr() + int(o), int(s)) for o, s in zip(offs[:-1], sizes)]
    h, d, s = _hash(torch, ctx, regions)
    host = big.cpu().numpy()
    exp = [orc.chunk_hashes(host[int(o):int(o) + int(sz)]) for o, sz in zip(offs[:-1], sizes)]
    assert np.array_equal(h, np.concatenate(exp))
    assert [int(x) for x in d] == [orc.region_digest(e) for e in exp]


def test_k1_full_2gib_region_and_digests(env):
    """c3-sized region at full size: every chunk hash and the region/snapshot
    digests (manifest of 256 KB: the digest kernel streams several stages)."""
    torch, kc, ctx, orc = env
    n = 2 * 2**30 + 12345
    buf = _rand_dev(torch, n, 11)
    small = _rand_dev(torch, 3 * CH + 7, 12)
    regions = sorted([(buf.data_ptr(), n), (small.data_ptr(), small.numel())])
    h, d, s = _hash(torch, ctx, regions, digests=True)
    hosts = {buf.data_ptr(): buf.cpu().numpy(), small.data_ptr(): small.cpu().numpy()}
    exp = [orc.chunk_hashes(hosts[b], threads=16) for b, _ in regions]
    assert np.array_equal(h, np.concatenate(exp))
    dig = [orc.region_digest(e) for e in exp]
    assert [int(x) for x in d] == dig
    assert s == orc.snapshot_digest([r[0] for r in regions], [r[1] for r in regions], dig)


def test_k1_zero_chunks_and_empty(env):
    torch, kc, ctx, orc = env
    z = torch.zeros(4 * CH, dtype=torch.uint8, device="cuda")
    h, _, _ = _hash(torch, ctx, [(z.data_ptr(), 4 * CH)], digests=False)
    assert all(int(x) == 0x5983DDA9F15715A4 for x in h)  # all-zero chunk value (SURVEY.md:930)
    h, d, s = _hash(torch, ctx, [], digests=True)
    assert h.size == 0


@pytest.mark.parametrize("groups_per_sm", [None, 1.0, 1.01, 2.5, 3.0, 3.02])
def test_k1_subwave_ring_boundaries(env, groups_per_sm):
    """The sub-wave warp-specialized ring (k1_hash_ws: 1-3 hashing warps per SM, 8 chunks per
    warp) and the switch to CpS above 3 x SMs chunk groups: chunk counts on each side of the
    HW = 1 / 2 / 3 boundaries, with ragged region tails (a 17-byte sub-stripe tail, a 20-byte
    region, a 100-byte one) that put the chunks in length-sorted order."""
    torch, kc, ctx, orc = env
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    C = 1 if groups_per_sm is None else int(round(groups_per_sm * sms)) * 8 + (5 if groups_per_sm % 1 else 0)
    tail = [CH + 17, 20, 100] if C >= 4 else []
    full = C - (2 + 1 + 1 if tail else 0)
    sizes = ([full * CH] if full else []) + tail
    offs = np.concatenate([[0], np.cumsum([(x + 255) // 256 * 256 for x in sizes])])
    big = _rand_dev(torch, int(offs[-1]), 4242 + C)
    regions = [(big.data_ptr() + int(o), int(x)) for o, x in zip(offs[:-1], sizes)]
    assert kc.count_chunks(regions) == C
    h, d, s = _hash(torch, ctx, regions)
    host = big.cpu().numpy()
    exp = [orc.chunk_hashes(host[int(o):int(o) + int(x)], threads=16) for o, x in zip(offs[:-1], sizes)]
    assert np.array_equal(h, np.concatenate(exp))
    dig = [orc.region_digest(e) for e in exp]
    assert [int(x) for x in d] == dig
    assert s == orc.snapshot_digest([r[0] for r in regions], [r[1] for r in regions], dig)


def test_k1_deterministic_across_calls(env):
    torch, kc, ctx, orc = env
    buf = _rand_dev(torch, 37 * CH + 5, 99)
    a = _hash(torch, ctx, [(buf.data_ptr(), buf.numel())])
    b = _hash(torch, ctx, [(buf.data_ptr(), buf.numel())])
    assert np.array_equal(a[0], b[0]) and a[2] == b[2]


@pytest.mark.parametrize("C", [1, 63, 64, 65, 1000, 4097])
def test_k3_written_set(env, C):
    torch, kc, ctx, orc = env
    rng = np.random.default_rng(C)
    pre = rng.integers(0, 2**63, size=C, dtype=np.int64)
    post = pre.copy()
    flip = rng.random(C) < 0.2
    flip[[0, C - 1]] = True
    post[flip] ^= 1
    dpre = torch.from_numpy(pre).cuda()
    dpost = torch.from_numpy(post).cuda()
    words = (C + 63) // 64
    bm = torch.zeros(words, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx.written(dpre.data_ptr(), dpost.data_ptr(), C, bm.data_ptr(), cnt.data_ptr())
    torch.cuda.synchronize()
    got = bm.cpu().numpy().view(np.uint64)
    exp = np.zeros(words, dtype=np.uint64)
    for k in np.nonzero(flip)[0]:
        exp[k // 64] |= np.uint64(1) << np.uint64(k % 64)
    assert np.array_equal(got, exp)
    assert int(cnt.item()) == int(flip.sum())
