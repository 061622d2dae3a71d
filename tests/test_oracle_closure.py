"""Pins for the oracle's O5 closure walker.

Lists are built so the expected outputs are closed forms: list i holds values
1..L (in list order) so the running sum at the j-th node is j(j+1)/2, and the
F1' mutation leaves 3v+1 in every node.
"""
import struct

import numpy as np
import pytest


def _build(n_lists, L, seed, nodes_base, heads_base, out_base, split_nodes=False):
    rng = np.random.default_rng(seed)
    n_nodes = n_lists * L
    slots = rng.permutation(n_nodes)
    nodes = bytearray(16 * n_nodes)
    heads = bytearray(8 * n_lists)
    expect_out = {}
    for i in range(n_lists):
        ss = slots[i * L:(i + 1) * L]
        for j, s in enumerate(ss):
            nxt = nodes_base + 16 * int(ss[j + 1]) if j + 1 < L else 0
            struct.pack_into("<QII", nodes, 16 * int(s), nxt, j + 1, 0)
            expect_out[int(s)] = (j + 1) * (j + 2) // 2
        struct.pack_into("<Q", heads, 8 * i, nodes_base + 16 * int(ss[0]))
    out = bytearray(8 * n_nodes)
    regions = [(heads_base, heads), (out_base, out)]
    if split_nodes:          # the node array spans two adjacent tracked regions
        half = 16 * (n_nodes // 2)
        regions += [(nodes_base, bytearray(nodes[:half])), (nodes_base + half, bytearray(nodes[half:]))]
    else:
        regions.append((nodes_base, nodes))
    return regions, expect_out


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("mutate", [False, True])
def test_walker_closed_form(orc, split, mutate):
    NB, HB, OB = 0x7F1200000000, 0x7F1200400000, 0x7F1200200000
    n_lists, L = 64, 5
    regions, expect = _build(n_lists, L, 1, NB, HB, OB, split_nodes=split)
    out_mem = [m for b, m in regions if b == OB][0]
    orc.walk_lists(regions, HB, n_lists, NB, OB, mutate=mutate)
    got = np.frombuffer(bytes(out_mem), dtype=np.uint64)
    for slot, v in expect.items():
        assert int(got[slot]) == v
    node_bytes = b"".join(bytes(m) for b, m in sorted(regions) if b >= NB and b < NB + 0x100000)
    vals = np.frombuffer(node_bytes, dtype=np.uint32).reshape(-1, 4)[:, 2]
    # values were 1..L per list; F1' rewrites them to 3v+1
    assert sorted(set(vals.tolist())) == ([3 * v + 1 for v in range(1, L + 1)] if mutate else list(range(1, L + 1)))


def test_walker_faults_outside_closure(orc):
    # PAPER.md:722-726 bound (3): a pointer the runtime never tracked is outside the closure
    NB, HB, OB = 0x7F1200000000, 0x7F1200400000, 0x7F1200200000
    regions, _ = _build(4, 3, 2, NB, HB, OB)
    heads = [m for b, m in regions if b == HB][0]
    struct.pack_into("<Q", heads, 8, 0x1000)          # untracked VA
    with pytest.raises(RuntimeError):
        orc.walk_lists(regions, HB, 4, NB, OB)


def test_walker_shifted_va_breaks(orc):
    # restoring at a different VA breaks the closure: relocate
    # the node region by 1 MiB without rewriting embedded pointers
    NB, HB, OB = 0x7F1200000000, 0x7F1200400000, 0x7F1200200000
    regions, _ = _build(8, 4, 3, NB, HB, OB)
    shifted = [(b + (0x100000 if b == NB else 0), m) for b, m in regions]
    with pytest.raises(RuntimeError):
        orc.walk_lists(shifted, HB, 8, NB, OB)


def test_cubin_module_vars_matches_readelf():
    """The oracle's ELF64 module-variable listing (F3) against binutils'
    readelf on the fixture code object: every defined, sized STT_OBJECT."""
    import shutil
    import subprocess
    from paper_2605_03208_b200 import build
    from oracle import snapshot
    import synth
    if not shutil.which("readelf"):
        pytest.skip("readelf not available")
    build.build_fixtures()
    out = subprocess.run(["readelf", "-s", "-W", synth.FIXTURE_CUBIN], capture_output=True, text=True).stdout
    exp = {}
    for line in out.splitlines():
        f = line.split()
        if len(f) >= 8 and f[3] == "OBJECT" and f[6] != "UND" and int(f[2]) > 0:
            exp[f[7]] = int(f[2])
    got = snapshot.cubin_module_vars(synth.FIXTURE_CUBIN)
    assert got == exp
    assert got == {"kc_fixture_cvals": 32, "kc_fixture_scale": 4, "kc_fixture_hits": 8}
