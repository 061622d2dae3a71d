"""CPU oracle for the Kerncap address-space-closure hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product path
(``paper_2605_03208_b200``) never imports, links or executes it, and this
package never imports the product path: the two share no code (the seeded
input generators live in ``synth/``, which holds none of the method's
arithmetic).

The arithmetic lives in ``oracle/kc_oracle.c`` (plain C, fp64, no FMA
contraction), loaded here through ctypes.  Each function cites the passage it
follows; the readings of the paper are DESIGN.md R1..R34.

Pins (what ties this oracle to something other than itself) are the
``-m "not gpu"`` tests in ``tests/test_oracle_*.py``.  Every function here is
pinned; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kc_oracle.c")
_LIB = os.path.join(_HERE, "libkc_oracle.so")

CHUNK = 65536  # hash/diff chunk, reading R1

# dtype codes, same numbering as the report contract (SURVEY.md 8(b) kc_dtype)
DT_BYTES, DT_U8, DT_I8, DT_U16, DT_I16, DT_U32, DT_I32, DT_U64, DT_I64, DT_F16, DT_BF16, DT_F32, DT_F64 = range(13)
DTYPE_NAMES = ["bytes", "u8", "i8", "u16", "i16", "u32", "i32", "u64", "i64", "f16", "bf16", "f32", "f64"]
ELEM_SIZE = [1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8]
FLOAT_DTYPES = (DT_F16, DT_BF16, DT_F32, DT_F64)

_build_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile kc_oracle.c with gcc (plain C11, -ffp-contract=off, no fast-math)."""
    with _build_lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call([
                "gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fno-strict-aliasing",
                "-Wall", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


class Report(ctypes.Structure):
    """O4 diff report."""
    _fields_ = [
        ("nbytes", ctypes.c_uint64), ("n_elems", ctypes.c_uint64), ("n_chunks", ctypes.c_uint64),
        ("differing_bytes", ctypes.c_uint64), ("differing_elems", ctypes.c_uint64), ("max_ulp", ctypes.c_uint64),
        ("max_abs", ctypes.c_double), ("max_rel", ctypes.c_double), ("percent_bytes", ctypes.c_double),
        ("nan_ref", ctypes.c_uint64), ("nan_act", ctypes.c_uint64), ("nan_pos_mismatch", ctypes.c_uint64),
        ("rel_undefined", ctypes.c_uint64), ("allclose_fail", ctypes.c_uint64),
        ("pass_", ctypes.c_int32), ("_pad", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_ if name != "_pad"}
        d["pass"] = d.pop("pass_")
        return d


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u8p = ctypes.c_void_p
        L.kco_xxh64.restype = ctypes.c_uint64
        L.kco_xxh64.argtypes = [u8p, ctypes.c_uint64, ctypes.c_uint64]
        L.kco_n_chunks.restype = ctypes.c_uint64
        L.kco_n_chunks.argtypes = [ctypes.c_uint64]
        L.kco_chunk_hashes.restype = None
        L.kco_chunk_hashes.argtypes = [u8p, ctypes.c_uint64, u8p]
        L.kco_region_digest.restype = ctypes.c_uint64
        L.kco_region_digest.argtypes = [u8p, ctypes.c_uint64, u8p]
        L.kco_snapshot_digest.restype = ctypes.c_uint64
        L.kco_snapshot_digest.argtypes = [u8p, u8p, u8p, ctypes.c_uint64, u8p]
        L.kco_written_set.restype = None
        L.kco_written_set.argtypes = [u8p, u8p, ctypes.c_uint64, u8p]
        L.kco_diff.restype = ctypes.c_int
        L.kco_diff.argtypes = [u8p, u8p, ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                               ctypes.c_int, ctypes.POINTER(Report), u8p]
        L.kco_walk_lists.restype = ctypes.c_int
        L.kco_walk_lists.argtypes = [u8p, u8p, u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64]
        _lib = L
    return _lib


def _buf(a) -> np.ndarray:
    """View any bytes-like / ndarray as a C-contiguous uint8 array (no copy if possible)."""
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a)
        return a.view(np.uint8).reshape(-1)
    return np.frombuffer(bytes(a) if not isinstance(a, (bytearray, memoryview)) else a, dtype=np.uint8)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# --------------------------------------------------------------------------- O2
def xxh64(data, seed: int = 0) -> int:
    """XXH64 of ``data`` (SURVEY.md 8(c) O2, Appendix A constants)."""
    b = _buf(data)
    return int(lib().kco_xxh64(_ptr(b), b.size, seed))


def n_chunks(size: int) -> int:
    return int(lib().kco_n_chunks(size))


def chunk_hashes(data, threads: int = 1) -> np.ndarray:
    """h[k] = XXH64(chunk k, seed 0) for a region's bytes (O2; readings R1-R3).

    ``threads`` splits chunks across host threads (ctypes releases the GIL);
    results are identical for every thread count (a concatenation)."""
    b = _buf(data)
    n = n_chunks(b.size)
    out = np.zeros(n, dtype=np.uint64)
    if n == 0:
        return out
    if threads <= 1 or n < 2:
        lib().kco_chunk_hashes(_ptr(b), b.size, out.ctypes.data)
        return out
    per = (n + threads - 1) // threads

    def work(t):
        k0, k1 = t * per, min(n, (t + 1) * per)
        if k0 >= k1:
            return
        lo, hi = k0 * CHUNK, min(b.size, k1 * CHUNK)
        lib().kco_chunk_hashes(b.ctypes.data + lo, hi - lo, out.ctypes.data + 8 * k0)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def region_digest(h: np.ndarray) -> int:
    """D_r = XXH64(LE64(h[0]) || ... || LE64(h[n-1]), 0)  (O2; reading R4)."""
    h = np.ascontiguousarray(h, dtype=np.uint64)
    scratch = np.zeros(max(1, 8 * h.size), dtype=np.uint8)
    return int(lib().kco_region_digest(_ptr(h), h.size, scratch.ctypes.data))


def snapshot_digest(bases, sizes, digests) -> int:
    """S over regions sorted by ascending base (O2; readings R4, R25)."""
    order = np.argsort(np.asarray(bases, dtype=np.uint64), kind="stable")
    b = np.ascontiguousarray(np.asarray(bases, dtype=np.uint64)[order])
    s = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64)[order])
    d = np.ascontiguousarray(np.asarray(digests, dtype=np.uint64)[order])
    scratch = np.zeros(max(1, 24 * b.size), dtype=np.uint8)
    return int(lib().kco_snapshot_digest(_ptr(b), _ptr(s), _ptr(d), b.size, scratch.ctypes.data))


# --------------------------------------------------------------------------- O3
def written_set(pre, post) -> np.ndarray:
    """W[k] = 1 iff chunk k's bytes differ between pre and post (O3)."""
    a, b = _buf(pre), _buf(post)
    if a.size != b.size:
        raise ValueError("pre/post sizes differ")
    w = np.zeros(n_chunks(a.size), dtype=np.uint8)
    if w.size:
        lib().kco_written_set(_ptr(a), _ptr(b), a.size, w.ctypes.data)
    return w


# --------------------------------------------------------------------------- O4
@dataclass
class DiffResult:
    report: dict
    bitmap: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))


def diff(ref, act, dtype: int = DT_BYTES, atol: float = 1e-8, rtol: float = 1e-5, equal_nan: bool = False,
         with_bitmap: bool = True) -> DiffResult:
    """O4 diff report of reference ``ref`` vs actual ``act`` (readings R8-R18)."""
    r, a = _buf(ref), _buf(act)
    if r.size != a.size:
        raise ValueError("ref/act sizes differ")
    rep = Report()
    nwords = (n_chunks(r.size) + 63) // 64
    bm = np.zeros(max(1, nwords), dtype=np.uint64)
    rc = lib().kco_diff(_ptr(r), _ptr(a), r.size, int(dtype), float(atol), float(rtol), int(bool(equal_nan)),
                        ctypes.byref(rep), bm.ctypes.data if with_bitmap else None)
    if rc != 0:
        raise ValueError(f"kco_diff: nbytes {r.size} not a multiple of element size {ELEM_SIZE[dtype]}")
    return DiffResult(rep.as_dict(), bm[:nwords])


# --------------------------------------------------------------------------- O5
def walk_lists(regions, heads_va: int, n_lists: int, nodes_base: int, out_va: int, mutate: bool = False,
               max_steps: int = 1 << 20):
    """Closure walker for fixture F1/F1'.

    ``regions``: list of (base_va, bytearray) -- modified in place (out, and
    nodes when ``mutate``).  Every VA is resolved through the region table."""
    regions = sorted(regions, key=lambda t: t[0])
    nreg = len(regions)
    bases = np.array([b for b, _ in regions], dtype=np.uint64)
    sizes = np.array([len(m) for _, m in regions], dtype=np.uint64)
    holders = [(ctypes.c_char * len(m)).from_buffer(m) for _, m in regions]
    ptrs = (ctypes.c_void_p * nreg)(*[ctypes.addressof(h) for h in holders])
    rc = lib().kco_walk_lists(bases.ctypes.data, sizes.ctypes.data, ctypes.addressof(ptrs), nreg, heads_va,
                              n_lists, nodes_base, out_va, int(mutate), max_steps)
    del holders
    if rc != 0:
        raise RuntimeError("closure walker fault: a VA outside every captured region (PAPER.md:712-726)")
    return regions
