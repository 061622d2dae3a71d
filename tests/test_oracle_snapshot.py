"""Pins for the O1 snapshot checker (oracle/snapshot.py: load, verify,
post_state, verify_sequence) -- CPU only.

The directories are hand-built by tests/snapshot_fixture.py from hand-chosen
bytes with oracle/ and numpy only (never by the product), in the paper's
capture layout (PAPER.md:681-697 [sec. 4.2.1], PAPER.md:937-953 [fig.
reproducer]) with the sentinel written last.  What pins the
checker to something other than itself:

* the fixture's hashes, digests and S (tests/golden/snapshot_fixture.txt) are
  re-derived here with python-xxhash, an independent XXH64;
* load/post_state return the hand-chosen bytes and fields the builder wrote
  (the post state is the builder's own post array, not an overlay);
* W is the hand-stated set of changed chunks;
* every corruption in snapshot_fixture.CORRUPTIONS / SEQ_CORRUPTIONS (sentinel
  missing, a manifest byte flipped, written idx or bin dropped, W off by one
  chunk, SHA-256 mismatch, overlapping regions, broken chain identity, ...)
  must raise, and the untouched fixture must verify.
"""
import os
import struct

import numpy as np
import pytest
import xxhash

import snapshot_fixture as F
from oracle import snapshot as S

CHUNK = 65536


def _x(b: bytes) -> int:
    return xxhash.xxh64_intdigest(b, seed=0)


def _lib_manifest(b: np.ndarray) -> list:
    return [_x(b[k * CHUNK:(k + 1) * CHUNK].tobytes()) for k in range((b.size + CHUNK - 1) // CHUNK)]


def _lib_digest(hs: list) -> int:
    return _x(b"".join(struct.pack("<Q", h) for h in hs))


@pytest.fixture
def pre_w(tmp_path):
    d = str(tmp_path / "snap")
    info = F.write_snapshot(d, F.fixture_regions(), "pre_w")
    return d, info


# --------------------------------------------------------------------------- golden
def test_golden_fixture_values_match_python_xxhash():
    """Every line of the golden file, re-derived from the hand-chosen bytes with
    python-xxhash (not the oracle) -- and the builder still produces them."""
    rows = [ln.split() for ln in open(F.GOLDEN) if ln.strip() and not ln.startswith("#")]
    regs = {r["base"]: r for r in F.fixture_regions()}
    digs = {}
    n = 0
    for row in rows:
        kind = row[0]
        if kind in ("chunk", "post_chunk"):
            r = regs[int(row[1], 16)]
            b = r["pre"] if kind == "chunk" else r["post"]
            k = int(row[2])
            assert int(row[3], 16) == _x(b[k * CHUNK:(k + 1) * CHUNK].tobytes()), row
        elif kind in ("digest", "post_digest"):
            r = regs[int(row[1], 16)]
            b = r["pre"] if kind == "digest" else r["post"]
            assert int(row[2], 16) == _lib_digest(_lib_manifest(b)), row
            if kind == "digest":
                digs[int(row[1], 16)] = int(row[2], 16)
        elif kind == "written":
            r = regs[int(row[1], 16)]
            expect = [k for k in range((r["pre"].size + CHUNK - 1) // CHUNK)
                      if r["pre"][k * CHUNK:(k + 1) * CHUNK].tobytes() != r["post"][k * CHUNK:(k + 1) * CHUNK].tobytes()]
            assert (row[2:] if row[2] != "-" else []) == [str(k) for k in expect], row
        elif kind == "S":
            blob = b"".join(struct.pack("<QQQ", b, regs[b]["pre"].size, digs[b]) for b in sorted(digs))
            assert int(row[1], 16) == _x(blob)
        n += 1
    assert n == len(rows) and any(r[0] == "S" for r in rows)
    assert F.golden_lines() == [" ".join(r) for r in rows]


def test_hand_stated_written_sets():
    """W by the fixture's construction: A chunks 1 and 3 (short), B none, C chunk 0
    (chunk 1 rewritten with identical bytes is not written)."""
    regs = F.fixture_regions()
    import oracle
    assert np.nonzero(oracle.written_set(regs[0]["pre"], regs[0]["post"]))[0].tolist() == [1, 3]
    assert np.nonzero(oracle.written_set(regs[1]["pre"], regs[1]["post"]))[0].tolist() == []
    assert np.nonzero(oracle.written_set(regs[2]["pre"], regs[2]["post"]))[0].tolist() == [0]


# --------------------------------------------------------------------------- load / post_state / verify
def test_load_returns_the_hand_built_fields(pre_w):
    d, info = pre_w
    snap = S.load(d)
    regs = F.fixture_regions()
    assert [(r.base, r.size, r.kind, r.status) for r in snap.regions] == \
        [(r["base"], r["pre"].size, r["kind"], "ok") for r in regs]
    assert [r.written.tolist() for r in snap.regions] == [[1, 3], [], [0]]
    assert [r.n_chunks for r in snap.regions] == [4, 1, 2]
    assert snap.dispatch["mode"] == "pre_w" and snap.dispatch["mangled_symbol"] == F.SYMBOL
    for r, e in zip(snap.regions, regs):
        assert np.array_equal(snap.region_bytes(r), e["pre"])


def test_post_state_equals_the_hand_built_post_bytes(pre_w):
    d, _ = pre_w
    snap = S.load(d)
    for r, e in zip(snap.regions, F.fixture_regions()):
        assert np.array_equal(snap.post_state(r), e["post"])


def test_verify_accepts_pre_w_and_reports_hand_stated_totals(pre_w):
    d, info = pre_w
    summ = S.verify(S.load(d))
    assert summ == {"regions": 3, "ok": 3, "written_chunks": 3, "snapshot_digest": info["S"], "module_vars": 0}


def test_verify_accepts_post_mode(tmp_path):
    d = str(tmp_path / "post")
    info = F.write_snapshot(d, F.fixture_regions(), "post")
    snap = S.load(d)
    for r, e in zip(snap.regions, F.fixture_regions()):
        assert np.array_equal(snap.post_state(r), e["post"])   # POST: the file is the post state
    assert S.verify(snap)["snapshot_digest"] == info["S"]


def test_partial_snapshot_s_covers_ok_regions_only(tmp_path):
    """R19 / PAPER.md:753-761: a region freed after the dispatch is "failed"; S covers the
    others.  An S that still includes the failed region (the advisor's finding against
    the product) must be rejected."""
    regs = F.fixture_regions()
    d = str(tmp_path / "partial")
    info = F.write_snapshot(d, regs, "pre_w", failed=(regs[2]["base"],))
    summ = S.verify(S.load(d))
    assert summ["ok"] == 2 and summ["written_chunks"] == 2
    s_ok = _x(b"".join(struct.pack("<QQQ", r["base"], r["pre"].size, _lib_digest(_lib_manifest(r["pre"])))
                       for r in regs[:2]))
    assert summ["snapshot_digest"] == info["S"] == s_ok
    s_all = _x(b"".join(struct.pack("<QQQ", r["base"], r["pre"].size, _lib_digest(_lib_manifest(r["pre"])))
                        for r in regs))
    F._edit_json(os.path.join(d, "capture_log.json"), lambda j: j.__setitem__("snapshot_digest", f"{s_all:016x}"))
    with pytest.raises(S.SnapshotError, match="snapshot digest"):
        S.verify(S.load(d))


@pytest.mark.parametrize("name", sorted(F.CORRUPTIONS))
def test_every_corruption_is_rejected(pre_w, name):
    d, _ = pre_w
    S.verify(S.load(d))               # the untouched fixture verifies
    F.CORRUPTIONS[name](d)
    with pytest.raises(S.SnapshotError):
        S.verify(S.load(d))


# --------------------------------------------------------------------------- sequences
def test_verify_sequence_accepts_and_recomputes_deps(tmp_path):
    d = str(tmp_path / "seq")
    info = F.write_sequence(d)
    summ = S.verify_sequence(d)
    assert summ["deps"] == info["deps"] == [[0, 0], [S.DEP_RAW | S.DEP_WAR, 0]]
    assert summ["written_chunks"] == [3, 1]


@pytest.mark.parametrize("name", sorted(F.SEQ_CORRUPTIONS))
def test_every_sequence_corruption_is_rejected(tmp_path, name):
    d = str(tmp_path / "seq")
    F.write_sequence(d)
    S.verify_sequence(d)
    F.SEQ_CORRUPTIONS[name](d)
    with pytest.raises(S.SnapshotError):
        S.verify_sequence(d)


def test_broken_chain_leaves_each_step_valid(tmp_path):
    """The chain corruption keeps both steps individually valid, so only the chain
    identity can reject it."""
    d = str(tmp_path / "seq")
    F.write_sequence(d)
    F.SEQ_CORRUPTIONS["broken_chain_identity"](d)
    for sub in ("step_000", "step_001"):
        S.verify(S.load(os.path.join(d, sub)))
    with pytest.raises(S.SnapshotError, match="after step 0 != before step 1"):
        S.verify_sequence(d)
