"""Pins for the oracle's O2 (XXH64, chunk manifest, digests) and O3 (written set).

Each pin ties the oracle to something other than itself: the published xxhsum
vectors (tests/golden/xxh64_vectors.txt), an independent library
(python-xxhash 3.7.0), closed forms, and brute force.
"""
import os
import struct

import numpy as np
import pytest
import xxhash

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _gen_v06(n):
    g, out = 2654435761, bytearray()
    for _ in range(n):
        out.append(g >> 24)
        g = (g * g) & 0xFFFFFFFF
    return bytes(out)


def _gen_v08(n):
    g, out = 2654435761, bytearray()
    for _ in range(n):
        out.append(g >> 56)
        g = (g * 11400714785074694797) & 0xFFFFFFFFFFFFFFFF
    return bytes(out)


def _golden_vectors():
    rows = []
    with open(os.path.join(GOLDEN, "xxh64_vectors.txt")) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            gen, length, seed, expect, prov = line.split()
            rows.append((gen, int(length), int(seed), int(expect, 16), prov))
    return rows


@pytest.mark.parametrize("gen,length,seed,expect,prov", _golden_vectors())
def test_xxh64_published_vectors(orc, gen, length, seed, expect, prov):
    if gen == "literal:":
        buf = b""
    elif gen == "v06":
        buf = _gen_v06(101)[:length]
    elif gen == "v08":
        buf = _gen_v08(2367)[:length]
    else:
        buf = bytes(length)
    assert orc.xxh64(buf, seed) == expect


def test_xxh64_short_strings(orc):
    # "a" and "abc" at seed 0
    assert orc.xxh64(b"a") == 0xD24EC4F1A98C6E5B
    assert orc.xxh64(b"abc") == 0x44BC2CF5AD770999


EDGE_LENGTHS = [0, 1, 3, 4, 5, 7, 8, 9, 11, 12, 15, 16, 17, 24, 31, 32, 33, 35, 36, 39, 40, 63, 64, 65,
                95, 96, 97, 127, 128, 129, 1000, 4095, 4096, 65535, 65536, 65537]


@pytest.mark.parametrize("seed", [0, 1, 2654435761, 0xFFFFFFFFFFFFFFFF])
def test_xxh64_differential_vs_library(orc, seed):
    rng = np.random.default_rng(7)
    lengths = EDGE_LENGTHS + list(rng.integers(0, 3000, size=60))
    for n in lengths:
        buf = rng.integers(0, 256, size=int(n), dtype=np.uint8).tobytes()
        assert orc.xxh64(buf, seed) == xxhash.xxh64_intdigest(buf, seed), n


def test_zero_chunk_value(orc):
    # all-zero 64 KiB chunk (SURVEY.md:930, library-computed)
    assert orc.xxh64(bytes(65536)) == 0x5983DDA9F15715A4


@pytest.mark.parametrize("size", [0, 1, 31, 32, 65535, 65536, 65537, 3 * 65536, 3 * 65536 + 17, 1 << 20])
def test_chunk_manifest_closed_form_and_library(orc, size):
    rng = np.random.default_rng(size)
    data = rng.integers(0, 256, size=size, dtype=np.uint8).tobytes()
    h = orc.chunk_hashes(data)
    assert len(h) == (size + 65535) // 65536               # n_r = ceil(size / 65536)
    for k in range(len(h)):
        piece = data[k * 65536:min(size, (k + 1) * 65536)]   # last chunk short, no padding (R3)
        assert int(h[k]) == xxhash.xxh64_intdigest(piece, 0)


def test_chunk_manifest_threads_identical(orc):
    rng = np.random.default_rng(3)
    data = rng.integers(0, 256, size=37 * 65536 + 1234, dtype=np.uint8)
    assert np.array_equal(orc.chunk_hashes(data, threads=1), orc.chunk_hashes(data, threads=5))


def test_region_and_snapshot_digest_vs_library(orc):
    rng = np.random.default_rng(11)
    h = rng.integers(0, 2**63, size=9, dtype=np.uint64) * 2 + 1
    le = b"".join(struct.pack("<Q", int(x)) for x in h)
    assert orc.region_digest(h) == xxhash.xxh64_intdigest(le, 0)
    assert orc.region_digest(np.zeros(0, dtype=np.uint64)) == xxhash.xxh64_intdigest(b"", 0)
    bases = [0x7F0000200000, 0x7F0000000000, 0x7F0000400000]
    sizes = [4096, 65536 * 3 + 5, 1]
    digs = [int(x) for x in h[:3]]
    # regions in ascending base order (R25) regardless of the order given
    order = np.argsort(bases)
    blob = b"".join(struct.pack("<QQQ", bases[i], sizes[i], digs[i]) for i in order)
    assert orc.snapshot_digest(bases, sizes, digs) == xxhash.xxh64_intdigest(blob, 0)


@pytest.mark.parametrize("size", [1, 65536, 65537, 5 * 65536 - 3])
def test_written_set_brute_force(orc, size):
    rng = np.random.default_rng(size + 1)
    pre = rng.integers(0, 256, size=size, dtype=np.uint8)
    post = pre.copy()
    nck = (size + 65535) // 65536
    flips = sorted(set([0, size - 1] + list(rng.integers(0, size, size=3))))
    for off in flips:
        post[off] ^= 0x5A
    expect = np.zeros(nck, dtype=np.uint8)
    for off in flips:
        expect[off // 65536] = 1
    assert np.array_equal(orc.written_set(pre, post), expect)
    assert not orc.written_set(pre, pre).any()
