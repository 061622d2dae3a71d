"""F4 multi-kernel capture
on the GPU, checked against the oracle.

Sequence (dependent and independent steps):
  step 0  kc_fixture_walk, mutate=1   (writes out; rewrites every node value)
  step 1  kc_fixture_axpy_u32         (y = 7x + y; touches neither list)
  step 2  kc_fixture_walk, mutate=0   (reads the rewritten nodes; writes out)
Hand-derived dependencies (include/kc.h KC_DEP_*, R33): step 2 on
step 0 is RAW (its nodes/out pointer parameters point into regions step 0
wrote), WAW (both write every out chunk) and WAR (step 0's out pointer lies in
a region step 2 writes); step 1 is independent of both.
"""
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_Y = 200_003          # u32 elements of x and y: 13 chunks, ragged tail
A = 7


def _up(synth, va, arr):
    import torch
    synth.dev_view(va, arr.nbytes).copy_(torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8).reshape(-1)))
    torch.cuda.synchronize()


def _down(synth, va, n):
    return synth.dev_view(va, n).cpu().numpy().copy()


@pytest.fixture(scope="module")
def env():
    import torch

    import oracle
    import synth
    from paper_2605_03208_b200 import build, kc
    build.build()
    oracle.build()
    torch.cuda.set_device(0)
    ctx = kc.Context(0)
    yield ctx, kc, synth, oracle
    ctx.close()


def _setup(env):
    ctx, kc, synth, oracle = env
    sizes = [s.size for s in synth.C1_SPECS] + [4 * N_Y, 4 * N_Y]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va, x_va, y_va = vas
    init = list(synth.c1_fill(nodes_va))
    rng = np.random.default_rng(synth.seed(1, 5))
    init += [rng.integers(0, 2**32, N_Y, dtype=np.uint64).astype(np.uint32).view(np.uint8),
             rng.integers(0, 2**32, N_Y, dtype=np.uint64).astype(np.uint32).view(np.uint8)]
    for va, arr in zip(vas, init):
        _up(synth, va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    walk = dict(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1))
    disp = [dict(walk, kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=1)),
            dict(image=image, mangled="kc_fixture_axpy_u32", grid=((N_Y + 255) // 256, 1, 1), block=(256, 1, 1),
                 kernarg=struct.pack("<QQII", x_va, y_va, N_Y, A)),
            dict(walk, kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=0))]
    return vas, sizes, init, disp


def _oracle_final(env, vas, sizes, init):
    """Expected state after the three steps: the O5 walker (mutate, then plain)
    and u32 arithmetic for the axpy step."""
    ctx, kc, synth, oracle = env
    nodes_va, heads_va, out_va = vas[:3]
    regs = [(va, bytearray(a.tobytes())) for va, a in zip(vas[:3], init[:3])]
    oracle.walk_lists(regs, heads_va, synth.C1_N_LISTS, nodes_va, out_va, mutate=True)
    oracle.walk_lists(regs, heads_va, synth.C1_N_LISTS, nodes_va, out_va, mutate=False)
    st = {va: np.frombuffer(bytes(m), dtype=np.uint8) for va, m in regs}
    x = init[3].view(np.uint32).astype(np.uint64)
    y = init[4].view(np.uint32).astype(np.uint64)
    st[vas[4]] = ((A * x + y) % 2**32).astype(np.uint32).view(np.uint8)
    st[vas[3]] = init[3]
    return st


def test_sequence_capture_deps_save_and_joint_replay(env, tmp_path):
    ctx, kc, synth, oracle = env
    from oracle import snapshot
    vas, sizes, init, disp = _setup(env)
    regions = sorted(zip(vas, sizes))
    seq, reps = ctx.capture_seq(disp, regions=regions)
    assert len(seq) == 3
    live = {va: _down(synth, va, sz) for va, sz in zip(vas, sizes)}
    exp = _oracle_final(env, vas, sizes, init)
    for va in vas:
        assert np.array_equal(live[va], exp[va]), f"the captured run itself != oracle at {va:x}"
    # written sets: step 0 = out (5 chunks) + nodes (10), step 1 = y (13), step 2 = out (5)
    assert [r["written_chunks"] for r in reps] == [15, 13, 5]
    # incremental steps copy only what the previous step changed
    assert reps[1]["d2h_bytes"] < sum(sizes) and reps[2]["d2h_bytes"] < sum(sizes)
    RAW, WAW, WAR = kc.KC_DEP_RAW, kc.KC_DEP_WAW, kc.KC_DEP_WAR
    expect = [[0, 0, 0], [0, 0, 0], [RAW | WAW | WAR, 0, 0]]
    assert seq.deps() == expect
    d = str(tmp_path / "seq")
    seq.save(d)
    summ = snapshot.verify_sequence(d)           # O1 per step + chain identity + deps from the files
    assert summ["deps"] == expect and summ["written_chunks"] == [15, 13, 5]

    for va in vas:
        ctx.free(va)
    steps, r = ctx.replay_seq(seq, keep=True)
    assert [s["pass"] for s in steps] == [1, 1, 1], steps
    assert [s["unexpected_chunks"] for s in steps] == [0, 0, 0]
    assert [s["inherited_chunks"] for s in steps] == [0, 0, 0]
    assert sorted((x.base, x.size) for x in r.regions()) == regions      # same VAs
    for va, sz in zip(vas, sizes):
        assert np.array_equal(_down(synth, va, sz), exp[va]), f"joint replay != oracle at {va:x}"
    r.release()

    # replay from the middle: the state before step 2 already holds step 0's rewrite
    steps, r = ctx.replay_seq(seq, first=2, count=1, keep=True)
    assert steps[0]["pass"] == 1
    assert np.array_equal(_down(synth, vas[2], sizes[2]), exp[vas[2]])
    r.release()

    # a modified step 0 (KC_VARIANT_DELTA=1: sums and rewrite both +1): step 0 fails,
    # the independent step 1 passes, and step 2 -- RAW-dependent on step 0 -- inherits it
    mod = open(os.path.join(os.path.dirname(synth.FIXTURE_CUBIN), "kc_fixtures_modified.cubin"), "rb").read()
    steps, _ = ctx.replay_seq(seq, overrides=[mod, None, None])
    assert [s["pass"] for s in steps] == [0, 1, 0], steps
    assert steps[0]["w"]["differing_bytes"] > 0 and steps[2]["w"]["differing_bytes"] > 0
    assert steps[1]["w"]["differing_bytes"] == 0 and steps[1]["unexpected_chunks"] == 0
    # divergence carried into each step: none into step 0; nodes (10 chunks) + out (5) into steps 1 and 2
    assert [s["inherited_chunks"] for s in steps] == [0, 15, 15]
    assert [s["unexpected_chunks"] for s in steps] == [0, 0, 0]
    # step 2's report is exactly the byte diff of its W chunks vs the captured post bytes
    # (the oracle's O4 on the out region: every node's running sum moved)
    assert steps[2]["w"]["differing_bytes"] == oracle.diff(exp[vas[2]], _mod_out(env, vas, init)).report["differing_bytes"]
    seq.free()


def _mod_out(env, vas, init):
    """out after the modified step 0 and the captured step 2, by the O5 walker:
    the rewrite is 3v+2, then plain running sums."""
    ctx, kc, synth, oracle = env
    nodes_va, heads_va, out_va = vas[:3]
    regs = [(va, bytearray(a.tobytes())) for va, a in zip(vas[:3], init[:3])]
    oracle.walk_lists(regs, heads_va, synth.C1_N_LISTS, nodes_va, out_va, mutate=True)
    nodes = np.frombuffer(bytes(regs[0][1]), dtype=[("next", "<u8"), ("value", "<u4"), ("pad", "<u4")]).copy()
    nodes["value"] = (nodes["value"].astype(np.uint64) + 1).astype(np.uint32)   # 3v+1 -> 3v+2
    regs[0] = (nodes_va, bytearray(nodes.tobytes()))
    oracle.walk_lists(regs, heads_va, synth.C1_N_LISTS, nodes_va, out_va, mutate=False)
    return np.frombuffer(bytes(regs[2][1]), dtype=np.uint8)


def test_sequence_host_arenas_and_bad_range(env):
    ctx, kc, synth, oracle = env
    vas, sizes, init, disp = _setup(env)
    seq, reps = ctx.capture_seq(disp[:2], regions=sorted(zip(vas, sizes)), host=True)
    assert seq.step(0).is_host() and seq.step(1).is_host()
    with pytest.raises(kc.KcError):
        ctx.replay_seq(seq, first=1, count=2)           # past the end
    for va in vas:
        ctx.free(va)
    steps, _ = ctx.replay_seq(seq)
    assert [s["pass"] for s in steps] == [1, 1]
    seq.free()
