"""Dispatch-state closure details on the GPU: a kernel launched with more than
48 KiB of dynamic shared memory (the opt-in function attribute is part of the
dispatch's runtime state) is captured from its code object,
restored at the same VAs, replayed and validated bit-exactly; the expected
output is written from the kernel's definition with numpy."""
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PER_BLOCK = 24 * 1024          # u32 per block: 96 KiB of dynamic shared memory
BLOCKS = 40


@pytest.fixture(scope="module")
def env():
    import torch

    import synth
    from paper_2605_03208_b200 import build, kc
    build.build()
    torch.cuda.set_device(0)
    ctx = kc.Context(0)
    yield ctx, kc, synth
    ctx.close()


def test_large_dynamic_smem_capture_replay(env):
    import torch
    ctx, kc, synth = env
    n = PER_BLOCK * BLOCKS
    vin, vout = ctx.alloc(4 * n), ctx.alloc(4 * n)
    x = np.random.default_rng(synth.seed(1, 9)).integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    synth.dev_view(vin, 4 * n).copy_(torch.from_numpy(x.view(np.uint8)))
    synth.dev_view(vout, 4 * n).zero_()
    torch.cuda.synchronize()
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    snap, rep = ctx.capture_dev(image=image, mangled="kc_fixture_smem_reverse", grid=(BLOCKS, 1, 1),
                                block=(1024, 1, 1), smem=4 * PER_BLOCK, kernarg=struct.pack("<QQI", vin, vout, PER_BLOCK),
                                regions=sorted([(vin, 4 * n), (vout, 4 * n)]))
    expect = (x.reshape(BLOCKS, PER_BLOCK)[:, ::-1] ^ np.arange(BLOCKS, dtype=np.uint32)[:, None]).reshape(-1)
    got = synth.dev_view(vout, 4 * n).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, expect), "the captured dispatch did not run as defined"
    assert rep["written_chunks"] == (4 * n + 65535) // 65536
    ctx.free(vin)
    ctx.free(vout)
    r, _ = ctx.restore_dev(snap)
    ctx.replay(r)
    reps, unexpected = ctx.validate(r)
    assert unexpected == 0 and len(reps) == 1 and reps[0]["differing_bytes"] == 0
    assert np.array_equal(synth.dev_view(vout, 4 * n).cpu().numpy().view(np.uint32), expect)
    r.release()
    snap.free()


@pytest.mark.parametrize("mode", ["pre_w", "post"])
@pytest.mark.parametrize("fused", [True, False])
def test_device_capture_ragged_regions(env, tmp_path, fused, mode, monkeypatch):
    """K6 (fused hash + copy) on ragged regions: sizes 1 .. 3 chunks + 40 B,
    16-byte aligned inside one allocation, including sub-32-byte tails and
    regions shorter than one hash stripe.  The persisted snapshot is checked
    by the oracle's O1 reader (every manifest recomputed, bytes compared with
    what the regions held), with K6 and with the unfused K1 + copy path."""
    import torch

    from oracle import snapshot
    ctx, kc, synth = env
    if not fused:
        monkeypatch.setenv("KC_NO_FUSED_CAPTURE", "1")
    sizes = [1, 17, 31, 32, 33, 4096 + 3, 65535, 65536, 65536 + 7, 3 * 65536 + 40, 1 << 20]
    offs, o = [], 0
    for sz in sizes:
        offs.append(o)
        o = (o + sz + 16 + 15) // 16 * 16          # 16-byte aligned, gaps between regions
    g = torch.Generator(device="cuda").manual_seed(synth.seed(1, 11))
    buf = torch.randint(0, 256, (o,), dtype=torch.uint8, device="cuda", generator=g)
    base = buf.data_ptr()
    regions = [(base + of, sz) for of, sz in zip(offs, sizes)]
    before = buf.cpu().numpy().copy()
    # the dispatch: u32 axpy over the largest region's first 4096 words
    xy = base + offs[-1]
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    snap, rep = ctx.capture_dev(image=image, mangled="kc_fixture_axpy_u32", grid=(4, 1, 1), block=(256, 1, 1),
                                kernarg=struct.pack("<QQII", xy, xy + 4 * 4096, 1024, 3), regions=regions,
                                mode=kc.KC_MODE_PRE_W if mode == "pre_w" else kc.KC_MODE_POST)
    if mode == "post":            # the stored state is the post-dispatch one
        before = buf.cpu().numpy().copy()
    d = str(tmp_path / "snap")
    snap.save(d)
    snap.free()
    s = snapshot.load(d)
    summ = snapshot.verify(s)
    assert summ["ok"] == len(sizes)
    for r, of, sz in zip(sorted(s.regions, key=lambda r: r.base), offs, sizes):
        assert np.array_equal(s.region_bytes(r), before[of:of + sz]), f"stored bytes of region +{of} differ"
    assert rep["written_chunks"] == 1


def test_cluster_launch_capture_replay(env, tmp_path):
    """A dispatch launched with thread-block clusters (Blackwell cluster launch,
    CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION = 2): the cluster dims are part of the
    dispatch state.  They are recorded (dispatch.json "cluster"), the replay
    launches with them again, and the output -- cluster rank, cluster size and a
    neighbour's value read through distributed shared memory -- matches the
    definition and validates bit-exactly."""
    import json
    import os
    ctx, kc, synth = env
    n = 64
    vout = ctx.alloc(4 * n)
    synth.dev_view(vout, 4 * n).zero_()
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    disp = dict(image=image, mangled="kc_fixture_cluster", grid=(n, 1, 1), block=(32, 1, 1),
                kernarg=struct.pack("<Q", vout), regions=[(vout, 4 * n)], cluster=(2, 1, 1))
    snap, rep = ctx.capture_dev(**disp)
    b = np.arange(n, dtype=np.uint32)
    rank = b % 2
    peer = (b - rank + (rank + 1) % 2) * 7 + 1
    expect = (rank << 24) | (2 << 16) | (peer & 0xFFFF)
    got = synth.dev_view(vout, 4 * n).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, expect), "the cluster launch did not run as defined"
    d = str(tmp_path / "cl")
    snap.save(d)
    assert json.load(open(os.path.join(d, "dispatch.json")))["cluster"] == [2, 1, 1]
    ctx.free(vout)
    r, _ = ctx.restore_dev(snap)
    ctx.replay(r)
    reps, unexpected = ctx.validate(r)
    assert reps and reps[0]["differing_bytes"] == 0 and unexpected == 0
    assert np.array_equal(synth.dev_view(vout, 4 * n).cpu().numpy().view(np.uint32), expect)
    r.release()
    snap.free()


def test_cooperative_launch_capture_replay(env):
    """A cooperative launch (grid-wide sync) is dispatch state too: recorded
    (kc_dispatch.flags, dispatch.json "cooperative") and replayed with
    CU_LAUNCH_ATTRIBUTE_COOPERATIVE; the neighbour values read after grid.sync()
    match the definition and validate bit-exactly."""
    ctx, kc, synth = env
    n = 96
    vstage, vout = ctx.alloc(4 * n), ctx.alloc(4 * n)
    synth.dev_view(vstage, 4 * n).zero_()
    synth.dev_view(vout, 4 * n).zero_()
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    snap, _ = ctx.capture_dev(image=image, mangled="kc_fixture_coop", grid=(n, 1, 1), block=(64, 1, 1),
                              kernarg=struct.pack("<QQ", vstage, vout),
                              regions=sorted([(vstage, 4 * n), (vout, 4 * n)]), cooperative=True)
    b = np.arange(n, dtype=np.uint32)
    expect = (((b + 1) % n) * 13 + 5) ^ 0xA5A5
    assert np.array_equal(synth.dev_view(vout, 4 * n).cpu().numpy().view(np.uint32), expect)
    ctx.free(vstage)
    ctx.free(vout)
    r, _ = ctx.restore_dev(snap)
    ctx.replay(r)
    reps, unexpected = ctx.validate(r)
    assert reps and all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0
    assert np.array_equal(synth.dev_view(vout, 4 * n).cpu().numpy().view(np.uint32), expect)
    r.release()
    snap.free()
