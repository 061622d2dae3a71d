"""The address-space closure end to end on the GPU (configs c1, c2):
capture in one process, VA-faithful restore + replay + validate in a fresh
one, checked against the oracle (O1 snapshot checker, O5 closure walker).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "closure_worker.py")


def run(*args, env=None, timeout=300):
    e = dict(os.environ)
    if env:
        e.update(env)
    p = subprocess.run([sys.executable, WORKER, *args], capture_output=True, text=True, timeout=timeout, env=e)
    assert p.returncode == 0, f"worker {args} failed:\n{p.stdout}\n{p.stderr}"
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2605_03208_b200 import build
    import oracle
    build.build()
    oracle.build()


def _walker_prediction(snapdir, mutate):
    import oracle
    from oracle import snapshot
    snap = snapshot.load(snapdir)
    regs = sorted(snap.regions, key=lambda r: r.base)
    mem = [(r.base, bytearray(snap.region_bytes(r).tobytes())) for r in regs]
    ka = open(os.path.join(snapdir, "kernarg.bin"), "rb").read()
    import struct
    h, o, nb, nl, mu = struct.unpack("<QQQIi", ka)
    oracle.walk_lists(mem, h, nl, nb, o, mutate=bool(mu))
    return {b: np.frombuffer(bytes(m), dtype=np.uint8) for b, m in mem}, (h, o, nb)


@pytest.mark.parametrize("mutate", [False, True])
def test_c1_capture_restore_replay_validate(tmp_path, mutate):
    d = str(tmp_path / "cap")
    cap = run("capture-c1", d, "--mode", "pre_w", *(["--mutate"] if mutate else []))
    assert cap["rc"] == 0
    from oracle import snapshot
    summ = snapshot.verify(snapshot.load(d))          # O1: format, manifests, digests, W
    assert summ["ok"] == 3
    pred, (heads_va, out_va, nodes_va) = _walker_prediction(d, mutate)
    # the original dispatch equals the oracle's closure walk
    orig_out = np.load(str(tmp_path / "cap_orig_out.npy"))
    assert np.array_equal(orig_out, pred[out_va])
    if mutate:
        assert np.array_equal(np.load(str(tmp_path / "cap_orig_nodes.npy")), pred[nodes_va])
    res = run("replay", d)
    assert "restore" in res, res
    assert [tuple(x) for x in res["regions"]] == sorted((r.base, r.size) for r in snapshot.load(d).regions)
    assert res["restore"]["verify_mismatch_chunks"] == 0
    # validation: bit-exact against the captured post bytes, nothing else written
    assert res["validate"], "no written regions validated"
    for rep in res["validate"]:
        assert rep["differing_bytes"] == 0 and rep["pass"] == 1
    assert res["unexpected_chunks"] == 0
    # the replay's dump equals the walker's prediction (closure property)
    dump = res["dump"]
    got_out = np.fromfile(os.path.join(dump, "output", f"region_{out_va:x}.bin"), dtype=np.uint8)
    assert np.array_equal(got_out, pred[out_va])


def test_c1_post_mode_diverges_for_in_place_kernel(tmp_path):
    """Capture timing (reading R7): POST replays from the post state, so an
    in-place kernel (F1') cannot reproduce its original output; PRE_W can."""
    d = str(tmp_path / "post")
    cap = run("capture-c1", d, "--mode", "post", "--mutate")
    assert cap["rc"] == 0
    from oracle import snapshot
    snapshot.verify(snapshot.load(d))
    res = run("replay", d)
    bad = [r for r in res["validate"] if r["differing_bytes"] > 0]
    assert bad, "POST-mode replay of an in-place kernel should diverge"


def test_c1_replay_iterations_recopy(tmp_path):
    d = str(tmp_path / "it")
    run("capture-c1", d, "--mode", "pre_w", "--mutate")
    res = run("replay", d, "--iterations", "5")
    assert all(r["differing_bytes"] == 0 for r in res["validate"])
    assert res["replay"]["iterations"] == 5
    # without recopy the in-place kernel accumulates: iteration 5 != captured post state
    res2 = run("replay", d, "--iterations", "3", "--no-recopy")
    assert any(r["differing_bytes"] > 0 for r in res2["validate"])


def test_va_squat_aborts_and_rolls_back(tmp_path):
    """PAPER.md:1080-1082 "VA faithfulness is a hard requirement":
    with every captured window occupied, restore aborts with
    KC_ERR_VA_UNAVAILABLE, nothing is dispatched or left mapped and the ctx
    stays usable; the snapshot itself is intact, so a fresh process restores it."""
    d = str(tmp_path / "sq")
    run("capture-c1", d)
    res = run("replay", d, "--squat")
    assert "squat" in res, res
    assert res["restore_status"] == -6, res
    assert "hard requirement" in res["message"]
    assert res["squat_free"] == 0 and res["ctx_healthy_after_abort"]
    ok = run("replay", d)
    assert "restore" in ok, ok
    assert all(r["differing_bytes"] == 0 for r in ok["validate"])


def test_corrupted_region_file_is_localised(tmp_path):
    d = str(tmp_path / "cor")
    run("capture-c1", d)
    from oracle import snapshot
    s = snapshot.load(d)
    r = max(s.regions, key=lambda x: x.size)
    p = os.path.join(d, r.data_file)
    b = bytearray(open(p, "rb").read())
    b[3 * 65536 + 5] ^= 0xFF
    open(p, "wb").write(bytes(b))
    res = run("replay", d)
    assert res["restore_status"] == -10
    assert res["report"]["verify_mismatch_chunks"] == 1, res
    assert "1 restored chunk" in res["message"]


def test_round_trip_snapshot_restore_resnapshot(tmp_path):
    """O6: snapshot -> restore -> re-snapshot gives identical files, manifests and S."""
    d = str(tmp_path / "rt")
    run("capture-c1", d, "--mutate")
    d2 = str(tmp_path / "rt2")
    res = run("recapture", d, d2)
    assert res["rc"] == 0
    from oracle import snapshot
    a, b = snapshot.load(d), snapshot.load(d2)
    assert [(r.base, r.size, r.digest) for r in a.regions] == [(r.base, r.size, r.digest) for r in b.regions]
    for ra, rb in zip(a.regions, b.regions):
        assert np.array_equal(a.region_bytes(ra), b.region_bytes(rb))
    assert a.log["snapshot_digest"] == b.log["snapshot_digest"]
    snapshot.verify(b)


@pytest.mark.parametrize("mode", ["post", "pre_w"])
def test_region_freed_after_dispatch_is_tolerated(tmp_path, mode):
    """a buffer freed between completion and snapshot fails
    alone; metadata and the other regions stay intact.  In both
    modes the logged snapshot digest covers the surviving regions only (PRE_W
    took S before the dispatch, over all three), so the strict O1 checker
    accepts the KC_PARTIAL snapshot."""
    d = str(tmp_path / "fr")
    cap = run("capture-c1", d, "--mode", mode, "--free", "1")
    assert cap["rc"] == 1  # KC_PARTIAL
    from oracle import snapshot
    s = snapshot.load(d)
    st = {r.base: r.status for r in s.regions}
    assert st[cap["vas"][1]] == "failed"
    assert sum(v == "ok" for v in st.values()) == 2
    summ = snapshot.verify(s)
    assert summ["ok"] == 2
    assert int(cap["report"]["snapshot_digest"]) == summ["snapshot_digest"]
    assert json.load(open(os.path.join(d, "memory_regions.json")))  # written first, still parses


def test_restore_merges_a_window_straddling_span(tmp_path):
    """Two captured regions 24 MiB apart, the second starting inside the first's
    32 MiB VA window and ending past it: a fresh process restores both at their
    VAs (the window is released and one covering both reserved; R28a)."""
    d = str(tmp_path / "gap")
    cap = run("capture-gap", d)
    assert cap["rc"] == 0, cap
    g = cap["geom"]
    M = 1 << 20
    assert g["a_off"] == 2 * M and g["b_off"] == 28 * M      # B starts inside A's window, ends past it
    res = run("replay", d)
    assert "restore" in res, res
    assert [tuple(x) for x in res["regions"]] == [(g["A"], 2 * M), (g["B"], 8 * M)]
    assert all(r["differing_bytes"] == 0 for r in res["validate"])


def test_staging_pieces_follow_io_chunk(tmp_path):
    """the number of D2H copies follows KERNCAP_SNAPSHOT_CHUNK_BYTES."""
    d = str(tmp_path / "st")
    cap = run("capture-c1", d, "--io-chunk", str(4 * 65536), env={"KC_IO_THREADS": "1"})
    # c1 regions: 655,360 / 65,536 / 327,680 B at 256 KiB pieces -> 3 + 1 + 2 copies; W = the 5
    # chunks of `out` (320 KiB) gathered through a 256 KiB stage -> 2 more copies
    assert cap["report"]["dma_calls"] == 8
    # one I/O thread: staging high water <= depth (2) x io chunk (reading R26)
    assert cap["report"]["staging_high_water"] <= 2 * 4 * 65536


def test_c2_llama_shaped_capture_replay(tmp_path):
    d = str(tmp_path / "c2")
    cap = run("capture-c2", d)
    assert cap["rc"] == 0 and cap["report"]["n_regions"] == 21
    assert cap["report"]["total_bytes"] == 159_383_552
    from oracle import snapshot
    summ = snapshot.verify(snapshot.load(d))
    assert summ["written_chunks"] >= 1
    res = run("replay", d)
    assert all(r["differing_bytes"] == 0 for r in res["validate"]), res["validate"]
    assert res["unexpected_chunks"] == 0
    orig = np.load(str(tmp_path / "c2_orig_out.npy"))
    attn = cap["vas"]["attn_out"]
    got = np.fromfile(os.path.join(res["dump"], "output", f"region_{attn:x}.bin"), dtype=np.uint8)
    assert np.array_equal(got, orig)


def test_inprocess_restore_after_free(tmp_path):
    """Capture, free every region, restore in the same process at the same
    VAs, replay, validate (the bench's capture->replay latency path)."""
    d = str(tmp_path / "ip")
    res = run("inproc", d)
    assert res["rc"] == 0
    assert "restore" in res, res
    assert all(r["differing_bytes"] == 0 for r in res["validate"])
    assert res["unexpected_chunks"] == 0 and res["out_equal"]


def test_memalloc_regions_restore_exactly_or_abort(tmp_path):
    """cuMemAlloc regions below the driver's pooling threshold share driver-
    reserved VA: restore replays cuMemAlloc in capture order and must either
    land on the exact VAs or abort with KC_ERR_VA_UNAVAILABLE -- never relocate
    (PAPER.md:1080-1082, 1106-1108)."""
    d = str(tmp_path / "ipm")
    res = run("inproc", d, "--memalloc")
    assert res["rc"] == 0
    if "restore" in res:
        assert all(r["differing_bytes"] == 0 for r in res["validate"]) and res["out_equal"]
    else:
        assert res["restore_status"] == -6 and "hard requirement" in res["message"]


def test_replay_override_validate_variant(tmp_path):
    """The paper's validate-variant workflow:
    an unmodified recompile replays to zero differing bytes, a modified kernel to a
    nonzero diff localised to the output region; the original snapshot is intact."""
    import synth
    d = str(tmp_path / "var")
    cap = run("capture-c1", d)
    out_va = cap["vas"][2]
    same = run("replay", d, "--override", os.path.join(ROOT, "synth", "kc_fixtures_recompiled.cubin"))
    assert all(r["differing_bytes"] == 0 for r in same["validate"]) and same["unexpected_chunks"] == 0
    mod = run("replay", d, "--override", os.path.join(ROOT, "synth", "kc_fixtures_modified.cubin"),
              "--typed", f"{out_va:x}:{synth.C1_N_NODES * 8}:u64")
    bad = [r for r in mod["validate"] if r["differing_bytes"] > 0]
    assert len(bad) == 1 and bad[0]["nbytes"] == synth.C1_N_NODES * 8   # only `out` differs
    assert mod["unexpected_chunks"] > 0
    typed = mod["typed"][0]
    # every node's running sum is off by its position j+1 (delta 1 per node): max |A-R| = list length
    assert typed["differing_elems"] == synth.C1_N_NODES and typed["max_ulp"] == synth.C1_LIST_LEN
    assert typed["pass"] == 0


def test_typed_validation_of_a_float_output(tmp_path):
    """kc_validate with a typed f32 sub-range (F2 decode-attention output): exact replay -> pass."""
    d = str(tmp_path / "c2t")
    cap = run("capture-c2", d)
    attn = cap["vas"]["attn_out"]
    res = run("replay", d, "--typed", f"{attn:x}:{32 * 64 * 4}:f32")
    t = res["typed"][0]
    assert t["n_elems"] == 32 * 64 and t["differing_elems"] == 0 and t["pass"] == 1 and t["max_abs"] == 0.0


@pytest.mark.parametrize("mode,mutate,host", [("pre_w", True, False), ("post", False, False),
                                               ("pre_w", True, True), ("post", False, True)])
def test_device_snapshot_capture_restore_replay(tmp_path, mode, mutate, host):
    """F1: the snapshot lives in an HBM arena (or a pinned host
    arena, kc_capture_host); persisted with kc_snapshot_save it is a valid
    kc-snapshot/1 directory (oracle O1); restored at the same VAs from the arena
    three times in one process (R28d), the replay reproduces the original output."""
    d = str(tmp_path / "dev")
    os.makedirs(d, exist_ok=True)
    res = run("devsnap", d, "--mode", mode, "--cycles", "3", *(["--mutate"] if mutate else []),
              *(["--host"] if host else []))
    assert res["is_host"] == host
    for cyc in res["cycles"]:
        assert cyc["regions"] == res["cycles"][0]["regions"]
        assert cyc["out_equal"] and cyc["restore"]["verify_mismatch_chunks"] == 0
        assert all(r["differing_bytes"] == 0 for r in cyc["validate"]) and cyc["unexpected_chunks"] == 0
        assert cyc["typed"][0]["pass"] == 1
    from oracle import snapshot
    summ = snapshot.verify(snapshot.load(d))
    assert summ["ok"] == 3
    assert res["arena_bytes"] >= sum(s for _, s in res["regions"])
    assert [tuple(x) for x in res["regions"]] == sorted((v, s) for v, s in zip(res["vas"], [655360, 65536, 327680]))
    assert res["restore"]["verify_mismatch_chunks"] == 0
    assert res["out_equal"]
    assert all(r["differing_bytes"] == 0 for r in res["validate"]) and res["unexpected_chunks"] == 0
    assert res["typed"][0]["differing_elems"] == 0 and res["typed"][0]["pass"] == 1
    pred, (heads_va, out_va, nodes_va) = _walker_prediction(d, mutate)
    if mode == "pre_w":   # the PRE_W snapshot holds the inputs: the oracle's walk reproduces the output
        assert np.array_equal(np.load(str(tmp_path / "dev_orig_out.npy")), pred[out_va])


@pytest.mark.parametrize("mutate", [False, True])
def test_device_snapshot_restored_into_the_live_restore(tmp_path, mutate):
    """kc_restore_dev_into (the repeated-replay fast path): each cycle captures from the
    restored state and restores the new snapshot over the live restore's mappings; the
    restore puts back the pre-state (the zeroed output), the replay reproduces the output
    the capture observed (with the mutating walk the state moves on every cycle), validate
    is clean, and a snapshot of other regions is refused with KC_ERR_ARG."""
    d = str(tmp_path / "inplace")
    os.makedirs(d, exist_ok=True)
    res = run("devsnap-inplace", d, "--cycles", "3", *(["--mutate"] if mutate else []))
    assert len(res["cycles"]) == 3 and res["refused"]
    for cyc in res["cycles"]:
        assert cyc["regions"] == res["cycles"][0]["regions"]
        assert cyc["capture"]["written_chunks"] > 0
        assert cyc["restore"]["verify_mismatch_chunks"] == 0 and cyc["restore"]["mapped_bytes"] == 0
        assert cyc["restored_pre"] and cyc["out_equal"]
        assert all(r["differing_bytes"] == 0 for r in cyc["validate"]) and cyc["unexpected_chunks"] == 0


@pytest.mark.parametrize("host", [False, True])
def test_incremental_capture_shares_unchanged_chunks(tmp_path, host):
    """F2 incremental capture: against a full base, only the chunks whose
    stored-state hash changed are copied (here the 5 chunks of `out` the first
    dispatch wrote, plus the second capture's own W); the rest reference the base, which is freed before the
    incremental snapshot is persisted (oracle O1 checks every stored byte
    against its manifest) and restored at the same VAs."""
    d = str(tmp_path / "incr")
    os.makedirs(d, exist_ok=True)
    res = run("incr", d, *(["--host"] if host else []))
    nodes, heads, out = res["sizes"]
    # first capture: every region + W = the 5 out chunks; second: only out (changed by the
    # first dispatch) + its own W = the 10 node chunks the mutating dispatch rewrites
    assert res["rep0"]["written_chunks"] == 5 and res["bytes0"] == nodes + heads + out + out
    assert res["shared1"] == nodes + heads          # unchanged chunks are referenced, not copied
    assert res["rep1"]["written_chunks"] == 10
    assert res["bytes1"] == out + nodes and res["rep1"]["d2h_bytes"] == out + nodes
    from oracle import snapshot
    summ = snapshot.verify(snapshot.load(d))
    assert summ["ok"] == 3
    assert res["restore"]["verify_mismatch_chunks"] == 0 and res["out_equal"]
    assert all(r["differing_bytes"] == 0 for r in res["validate"]) and res["unexpected_chunks"] == 0
    assert res["typed"][0]["pass"] == 1


@pytest.mark.parametrize("cupti", [False, True])
def test_module_vars_capture_replay(tmp_path, cupti):
    """F3: the application sets __constant__ /
    __device__ variables of its own module; the capture records them (and,
    with the CUPTI hook, the code object from the module load), a fresh
    process restores them into the replay module, and the replay reproduces
    the output; without them (KC_NO_MODULE_VARS=1) it does not."""
    d = str(tmp_path / "mv")
    os.makedirs(d, exist_ok=True)
    cap = run("capture-modvar", d, *(["--cupti"] if cupti else []))
    assert cap["rc"] == 0
    mv = json.load(open(os.path.join(d, "module_vars.json")))
    byname = {v["name"]: v for v in mv["vars"]}
    assert {"kc_fixture_cvals", "kc_fixture_scale", "kc_fixture_hits"} <= set(byname)
    assert byname["kc_fixture_cvals"]["size"] == 32 and not byname["kc_fixture_cvals"]["written"]
    assert byname["kc_fixture_hits"]["written"]  # the dispatch counted itself
    hits = np.fromfile(os.path.join(d, byname["kc_fixture_hits"]["post"]), dtype=np.uint64)
    assert int(hits[0]) == 1000 + cap["n"]
    from oracle import snapshot
    summ = snapshot.verify(snapshot.load(d))
    assert summ["ok"] == 1 and summ["module_vars"] >= 3
    orig = np.load(str(tmp_path / "mv_orig_out.npy"))
    res = run("replay", d)
    assert res["replay"]["module_vars_restored"] >= 3
    assert res["modvars"][0] >= 3 and res["modvars"][1] == 0  # post values reproduced (hits too)
    assert all(r["differing_bytes"] == 0 for r in res["validate"]) and res["unexpected_chunks"] == 0
    out_file = os.path.join(res["dump"], "output", "region_%x.bin" % cap["out_va"])
    # (with the CUPTI hook the tracked region is the whole mapped VMM range, so compare the prefix)
    assert np.array_equal(np.fromfile(out_file, dtype=np.uint8)[:orig.size], orig)
    neg = run("replay", d, env={"KC_NO_MODULE_VARS": "1"})
    assert neg["replay"]["module_vars_restored"] == 0
    assert any(r["differing_bytes"] > 0 for r in neg["validate"])


@pytest.mark.parametrize("mutate", [False, True])
def test_published_device_snapshot_replays_in_another_process(tmp_path, mutate):
    """F1 across processes (kc_snapshot_publish): the region bytes stay in the
    capturing process's HBM and a fresh process restores them through CUDA IPC
    at the captured VAs (copy-in fused with the verify), replays and validates
    bit-exactly; its dump equals the oracle's closure walk over the normal
    (file) copy of the same snapshot.  Host and incremental snapshots are
    refused; once the publisher frees the snapshot a late restore fails
    cleanly (KC_ERR_STATE)."""
    import paper_2605_03208_b200.kc as kc
    from oracle import snapshot
    d = str(tmp_path / "pub")
    res = run("publish", d, *(["--mutate"] if mutate else []))
    assert res["refused"] == [kc.KC_ERR_STATE, kc.KC_ERR_STATE]
    # the publisher freed the snapshot at the end: the directory is revoked
    assert os.path.exists(os.path.join(d, "memory", "device_arena.revoked"))
    assert not any(f.endswith(".bin") for f in os.listdir(os.path.join(d, "memory")))
    files = d + "_files"
    assert snapshot.verify(snapshot.load(files))["ok"] == 3
    child = res["child"]
    assert res["child_rc"] == 0 and "restore" in child, child
    assert child["restore"]["verify_mismatch_chunks"] == 0
    assert child["restore"]["h2d_bytes"] == sum(s for _, s in child["regions"])
    assert [tuple(x) for x in child["regions"]] == sorted((r.base, r.size) for r in snapshot.load(files).regions)
    assert child["validate"] and all(r["differing_bytes"] == 0 and r["pass"] == 1 for r in child["validate"])
    assert child["unexpected_chunks"] == 0
    pred, (heads_va, out_va, nodes_va) = _walker_prediction(files, mutate)
    got = np.fromfile(os.path.join(child["dump"], "output", f"region_{out_va:x}.bin"), dtype=np.uint8)
    assert np.array_equal(got, pred[out_va])
    assert res["late"].get("restore_status") == kc.KC_ERR_STATE, res["late"]


def test_tampered_code_object_is_refused(tmp_path):
    """dispatch.json records the code object's SHA-256 (the paper matches HSACO
    blobs by SHA-256); the O1 checker recomputes it with
    hashlib, and a restore of a snapshot whose kernel.cubin was altered fails
    with KC_ERR_FORMAT before anything is mapped."""
    import hashlib
    import paper_2605_03208_b200.kc as kc
    from oracle import snapshot
    d = str(tmp_path / "cap")
    run("capture-c1", d)
    disp = json.load(open(os.path.join(d, "dispatch.json")))
    cub = os.path.join(d, "kernel.cubin")
    assert disp["code_object_sha256"] == hashlib.sha256(open(cub, "rb").read()).hexdigest()
    snapshot.verify(snapshot.load(d))
    b = bytearray(open(cub, "rb").read())
    b[len(b) // 2] ^= 0x40
    open(cub, "wb").write(bytes(b))
    res = run("replay", d)
    assert res.get("restore_status") == kc.KC_ERR_FORMAT, res


@pytest.mark.parametrize("mode", ["pre_w", "post"])
def test_interposed_capture_of_an_unmodified_application(tmp_path, mode):
    """A3 interposed mode: the application
    loads the module, allocates with cuMemAlloc and launches the list walk twice
    through the driver API; the CUPTI hook captures launch #1 (F1', in place).
    The application's launches each ran exactly once (its nodes hold 3v+1, not a
    double rewrite); the snapshot passes the O1 checker, holds only the three
    application allocations (none of the library's own), and a fresh process
    replays it bit-exactly (PRE_W) -- POST starts from the rewritten nodes, so
    its replay diverges exactly as R7 predicts."""
    import oracle
    from oracle import snapshot
    d = str(tmp_path / "ip")
    res = run("interpose", d, "--mode", mode)
    assert res["status"]["state"] == 3, res["status"]
    assert res["status"]["report"]["n_regions"] == 3 and res["status"]["report"]["written_chunks"] > 0
    assert sorted(res["ptrs"]) == sorted(b for b, _ in res["tracked"])
    snap = snapshot.load(d)
    snapshot.verify(snap)
    assert sorted(r.base for r in snap.regions) == sorted(res["ptrs"])
    # what the application saw: plain walk, then the in-place walk, each once
    init_nodes = np.load(str(tmp_path / "ip_init_nodes.npy"))
    nodes_dt = np.dtype([("next", "<u8"), ("value", "<u4"), ("pad", "<u4")])
    v0 = init_nodes.view(nodes_dt)["value"].astype(np.uint64)
    app_nodes = np.load(str(tmp_path / "ip_app_nodes.npy")).view(nodes_dt)
    assert np.array_equal(app_nodes["value"], ((3 * v0 + 1) % 2**32).astype(np.uint32))
    rep = run("replay", d)
    assert "restore" in rep, rep
    if mode == "pre_w":
        assert all(r["differing_bytes"] == 0 for r in rep["validate"]) and rep["unexpected_chunks"] == 0
    else:
        assert any(r["differing_bytes"] > 0 for r in rep["validate"])


def test_interposed_sequence_capture(tmp_path):
    """F4 from an unmodified application: kc_interpose_arm_seq captures three
    consecutive launches (walk with the in-place rewrite, an independent axpy,
    a walk reading the rewritten nodes).  The saved sequence passes the
    oracle's sequence checker (O1 per step, chain identity, deps from the
    files), the dependency matrix is the hand-derived one, and every step
    replays bit-exactly in a fresh process."""
    import paper_2605_03208_b200.kc as kc
    from oracle import snapshot
    d = str(tmp_path / "seq")
    res = run("interpose-seq", d)
    assert res["status"]["state"] == 3, res["status"]
    RAW, WAW, WAR = kc.KC_DEP_RAW, kc.KC_DEP_WAW, kc.KC_DEP_WAR
    expect = [[0, 0, 0], [0, 0, 0], [RAW | WAW | WAR, 0, 0]]
    assert res["deps"] == expect
    summ = snapshot.verify_sequence(d)
    assert summ["deps"] == expect and summ["written_chunks"][1] > 0
    for k in range(3):
        rep = run("replay", os.path.join(d, f"step_{k:03d}"))
        assert "restore" in rep, rep
        assert all(r["differing_bytes"] == 0 for r in rep["validate"]) and rep["unexpected_chunks"] == 0


def test_interposed_capture_of_a_triton_program(tmp_path):
    """A real JIT framework as the application: an unmodified Triton program
    (tests/apps/triton_app.py, no library code; its module load and
    cuLaunchKernel(Ex) go through the driver API) run by `cli capture`, which
    injects libkc.so with CUDA_INJECTION64_PATH and captures the second
    `scaled_add` launch.  The program's own result is intact, the snapshot passes
    the O1 checker and holds the code object Triton loaded, and `cli replay` in a
    fresh process validates bit-exactly."""
    pytest.importorskip("triton")
    from oracle import snapshot
    d = str(tmp_path / "tri")
    cli = [sys.executable, "-m", "paper_2605_03208_b200.cli"]
    p = subprocess.run(cli + ["capture", "--kernel", "scaled_add", "--index", "1", "--out", d, "--",
                              sys.executable, os.path.join(ROOT, "tests", "apps", "triton_app.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    lines = [json.loads(x) for x in p.stdout.strip().splitlines() if x.startswith("{")]
    assert lines[0]["out_ok"], "the application's own result is wrong: its launch must run exactly once"
    assert lines[-1]["captured"]
    snap = snapshot.load(d)
    snapshot.verify(snap)
    assert "scaled_add" in snap.dispatch["mangled_symbol"] and snap.dispatch["code_object_bytes"] > 0
    p = subprocess.run(cli + ["replay", d], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    rep = json.loads(p.stdout.strip().splitlines()[-1])
    assert rep["pass"] and rep["validate"] and all(r["differing_bytes"] == 0 for r in rep["validate"])


@pytest.mark.parametrize("host", [False, True])
def test_load_once_replay_many(tmp_path, host):
    """kc_snapshot_load: a fresh process loads the file snapshot into HBM (or
    pinned host memory) once, verified against its manifests, then restores at
    the captured VAs, replays and validates three times from memory."""
    d = str(tmp_path / "cap")
    run("capture-c1", d, "--mutate")
    res = run("load-replay", d, "--cycles", "3", *(["--host"] if host else []))
    assert res["is_host"] == host and len(res["cycles"]) == 3
    regs = res["cycles"][0]["regions"]
    for c in res["cycles"]:
        assert c["ok"] and c["verify"] == 0 and c["regions"] == regs


def test_saved_sequence_replays_in_a_fresh_process(tmp_path):
    """kc_seq_load: the interposed sequence (walk, axpy, walk) saved by one
    process is loaded and jointly replayed by another, every step bit-exact."""
    d = str(tmp_path / "seq")
    run("interpose-seq", d)
    res = run("load-seq", d)
    assert res["n"] == 3 and [s["pass"] for s in res["steps"]] == [1, 1, 1], res["steps"]
    import paper_2605_03208_b200.kc as kc   # the loaded steps keep their kernarg layouts: same dependencies
    assert res["deps"] == [[0, 0, 0], [0, 0, 0], [kc.KC_DEP_RAW | kc.KC_DEP_WAW | kc.KC_DEP_WAR, 0, 0]]
    assert [s["inherited_chunks"] for s in res["steps"]] == [0, 0, 0]


def test_cli_capture_of_an_application_without_kc_code(tmp_path):
    """The paper's workflow on CUDA (`kerncap capture` / `replay`):
    `python -m paper_2605_03208_b200.cli capture --kernel kc_fixture_walk --index 1
    --out DIR -- APP` runs a driver-API application that contains no library code.
    The driver loads libkc.so through CUDA_INJECTION64_PATH (InitializeInjection),
    whose CUPTI hook tracks the allocations and captures launch #1.  The
    application's own results are intact (each launch ran once), and `cli replay`
    in a fresh process validates bit-exactly; `cli info` summarises the snapshot."""
    from oracle import snapshot
    d = str(tmp_path / "cli")
    app_out = str(tmp_path / "app.npz")
    cli = [sys.executable, "-m", "paper_2605_03208_b200.cli"]
    p = subprocess.run(cli + ["capture", "--kernel", "kc_fixture_walk", "--index", "1", "--out", d, "--",
                              sys.executable, os.path.join(ROOT, "tests", "apps", "driver_app.py"), app_out, ROOT],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    assert json.loads(p.stdout.strip().splitlines()[-1])["captured"]
    app = np.load(app_out)
    nodes_dt = np.dtype([("next", "<u8"), ("value", "<u4"), ("pad", "<u4")])
    v0 = app["init_nodes"].view(nodes_dt)["value"].astype(np.uint64)
    assert np.array_equal(app["nodes"].view(nodes_dt)["value"], ((3 * v0 + 1) % 2**32).astype(np.uint32))
    snap = snapshot.load(d)
    snapshot.verify(snap)
    assert sorted(r.base for r in snap.regions) == sorted(int(x) for x in app["ptrs"])
    p = subprocess.run(cli + ["replay", d], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    rep = json.loads(p.stdout.strip().splitlines()[-1])
    print(f"cli replay: {rep.get('process_layouts')} process layout(s)")
    assert rep["pass"] and rep["unexpected_chunks"] == 0
    p = subprocess.run(cli + ["info", d], capture_output=True, text=True, timeout=120, cwd=ROOT)
    info = json.loads(p.stdout.strip().splitlines()[-1])
    assert info["kernel"] == "kc_fixture_walk" and info["regions"] == 3


def test_failed_interposed_capture_never_blocks_the_application(tmp_path):
    """Liveness: when the interposed capture fails (here:
    its snapshot cannot be written), the state says so with the error, and the
    application's launch still ran exactly once with correct results."""
    import paper_2605_03208_b200.kc as kc
    d = str(tmp_path / "ipbad")
    res = run("interpose", d, "--bad-dir")
    assert res["status"]["state"] == -1 and res["status"]["rc"] == kc.KC_ERR_IO, res["status"]
    init_nodes = np.load(str(tmp_path / "ipbad_init_nodes.npy"))
    nodes_dt = np.dtype([("next", "<u8"), ("value", "<u4"), ("pad", "<u4")])
    v0 = init_nodes.view(nodes_dt)["value"].astype(np.uint64)
    app_nodes = np.load(str(tmp_path / "ipbad_app_nodes.npy")).view(nodes_dt)
    assert np.array_equal(app_nodes["value"], ((3 * v0 + 1) % 2**32).astype(np.uint32))


def test_cli_sequence_capture_and_joint_replay(tmp_path):
    """`cli capture --count 3` on an application without library code captures
    its three dependent launches as a sequence (kc-sequence/1, saved when the
    last step completes); `cli replay-seq` in a fresh process replays them
    jointly, every step bit-exact, with the hand-derived dependency matrix."""
    import paper_2605_03208_b200.kc as kc
    from oracle import snapshot
    d = str(tmp_path / "cliseq")
    cli = [sys.executable, "-m", "paper_2605_03208_b200.cli"]
    p = subprocess.run(cli + ["capture", "--count", "3", "--out", d, "--", sys.executable,
                              os.path.join(ROOT, "tests", "apps", "driver_seq_app.py"), ROOT],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    RAW, WAW, WAR = kc.KC_DEP_RAW, kc.KC_DEP_WAW, kc.KC_DEP_WAR
    expect = [[0, 0, 0], [0, 0, 0], [RAW | WAW | WAR, 0, 0]]
    assert snapshot.verify_sequence(d)["deps"] == expect
    p = subprocess.run(cli + ["replay-seq", d], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["pass"] and res["n"] == 3 and res["deps"] == expect


def test_interposition_skips_launches_recorded_into_a_cuda_graph(tmp_path):
    """Stream capture records launches without running them: the hook neither
    counts nor captures them (a device sync would also invalidate the graph
    capture).  The graph still replays for the application, and launch #0 of
    the kernel is the first one that actually runs directly (mutate = 1)."""
    import struct
    from oracle import snapshot
    d = str(tmp_path / "graph")
    res = run("interpose-graph", d)
    assert res["seen_after_capture"] == 0 and res["status"]["state"] == 3, res
    assert res["mutated_once"]
    snap = snapshot.load(d)
    snapshot.verify(snap)
    ka = open(os.path.join(d, "kernarg.bin"), "rb").read()
    assert struct.unpack("<QQQIi", ka)[4] == 1      # the captured dispatch is the direct, mutating launch
