"""Pins for the oracle's F4 sequence checks (oracle/snapshot.py sequence_deps,
DESIGN.md R33): hand-built step descriptions whose dependency flags are fixed
by the definition, one flag at a time, plus the negative cases (a pointer
into an unwritten region, a scalar that happens to equal a VA but has a
4-byte slot, disjoint chunks of one region)."""
import struct

import numpy as np

from oracle import snapshot as S

A_BASE, B_BASE, C_BASE = 0x7F0000000000, 0x7F0000400000, 0x7F0000800000
SIZE = 4 << 20


def _step(tmp_path, name, params, written):
    """params: list of (value, size) kernel parameters; written: {region index: [chunks]}."""
    d = tmp_path / name
    d.mkdir()
    ka, layout, off = b"", [], 0
    for v, sz in params:
        off = (off + sz - 1) // sz * sz
        ka = ka.ljust(off, b"\0") + (struct.pack("<Q", v) if sz == 8 else struct.pack("<I", v & 0xFFFFFFFF))
        layout.append({"offset": off, "size": sz})
        off += sz
    (d / "kernarg.bin").write_bytes(ka)
    regs = []
    for i, b in enumerate((A_BASE, B_BASE, C_BASE)):
        r = S.SnapRegion(b, SIZE, "vmm", "ok", 0, "")
        r.written = np.array(sorted(written.get(i, [])), dtype=np.uint64)
        regs.append(r)
    return S.Snapshot(str(d), {"kernarg_layout": layout}, regs, {})


def test_raw_only(tmp_path):
    s0 = _step(tmp_path, "s0", [(A_BASE + 16, 8)], {1: [3]})           # reads A, writes B chunk 3
    s1 = _step(tmp_path, "s1", [(B_BASE + SIZE - 1, 8)], {2: [0]})      # points at B's last byte, writes C
    assert S.sequence_deps([s0, s1]) == [[0, 0], [S.DEP_RAW, 0]]


def test_waw_only_needs_the_same_chunk(tmp_path):
    s0 = _step(tmp_path, "s0", [], {0: [1, 2]})
    s1 = _step(tmp_path, "s1", [], {0: [2]})
    s2 = _step(tmp_path, "s2", [], {0: [5]})                            # same region, other chunk
    d = S.sequence_deps([s0, s1, s2])
    assert d[1][0] == S.DEP_WAW and d[2][0] == 0 and d[2][1] == 0


def test_war_only(tmp_path):
    s0 = _step(tmp_path, "s0", [(C_BASE, 8)], {})                      # reads C, writes nothing
    s1 = _step(tmp_path, "s1", [], {2: [7]})                            # overwrites C
    assert S.sequence_deps([s0, s1]) == [[0, 0], [S.DEP_WAR, 0]]


def test_non_pointers_are_ignored(tmp_path):
    s0 = _step(tmp_path, "s0", [], {0: [0]})
    # a 4-byte parameter cannot hold a VA; a pointer one past the end of A is not in A
    s1 = _step(tmp_path, "s1", [(A_BASE, 4), (A_BASE + SIZE, 8)], {})
    assert S.sequence_deps([s0, s1]) == [[0, 0], [0, 0]]


def test_all_three_and_lower_triangle(tmp_path):
    s0 = _step(tmp_path, "s0", [(A_BASE, 8)], {0: [0], 1: [0]})
    s1 = _step(tmp_path, "s1", [(B_BASE, 8)], {0: [0]})
    d = S.sequence_deps([s0, s1])
    assert d == [[0, 0], [S.DEP_RAW | S.DEP_WAW | S.DEP_WAR, 0]]
