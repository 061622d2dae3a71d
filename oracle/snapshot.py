"""O1: independent reader/checker of the kc-snapshot/1 directory -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s oracle legs use
this module; it never imports the product path (``paper_2605_03208_b200``).

Parses the capture directory with Python's json (not the product's C++
parser), checks every file's presence and length, recomputes every manifest,
digest and written set with the oracle's own XXH64 (oracle/kc_oracle.c), and
checks the sentinel.  The format is the paper's capture layout
(PAPER.md:681-697 [sec. 4.2.1 "chunked, VA-faithful snapshot": one file per
region named by its base VA, metadata before the bulk copy]; PAPER.md:937-953
[fig. reproducer, ``capture/``]) with the sentinel-last rule of SPEC.md:412-426,
as laid out in DESIGN.md section 3 (readings R1-R7, R19, R25).

Strictness (pins: tests/test_oracle_snapshot.py over hand-built directories):
every ``ok`` region must have its region file, its manifest, its post
manifest and its written-chunk index; PRE_W regions with a non-empty W must
have the written bytes; every length is checked; the post digests and
per-region written counts logged in ``capture_log.json`` are recomputed; the
snapshot digest S covers exactly the regions whose final status is ``ok``.
Any violation raises ``SnapshotError`` (an AssertionError, so it survives
``python -O``-free test runs and older callers alike).
"""
from __future__ import annotations

import hashlib
import json
import os
import re
from dataclasses import dataclass, field

import numpy as np

from . import CHUNK, chunk_hashes, n_chunks, region_digest, snapshot_digest


class SnapshotError(AssertionError):
    """A kc-snapshot/1 (or kc-sequence/1) directory violates the format."""


def _check(cond, msg: str):
    if not cond:
        raise SnapshotError(msg)


_HEX_RE = re.compile(r"^[0-9a-f]+$")
_DIG_RE = re.compile(r"^[0-9a-f]{16}$")


def _read_u64(path: str, what: str) -> np.ndarray:
    _check(os.path.isfile(path), f"{what}: {os.path.basename(path)} missing")
    n = os.path.getsize(path)
    _check(n % 8 == 0, f"{what}: {n} bytes is not a whole number of u64")
    return np.fromfile(path, dtype="<u8")


@dataclass
class SnapRegion:
    base: int
    size: int
    kind: str
    status: str
    digest: int
    data_file: str
    written: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))
    n_chunks: int = -1          # as recorded in memory_regions.json
    post_digest: int = -1       # as recorded in capture_log.json
    logged_written: int = -1    # capture_log.json written_chunks of this region
    has_idx: bool = False       # written/region_<hex>.idx present


@dataclass
class Snapshot:
    dir: str
    dispatch: dict
    regions: list
    log: dict

    def _hx(self, r: SnapRegion) -> str:
        return f"{r.base:x}"

    def region_bytes(self, r: SnapRegion) -> np.ndarray:
        p = os.path.join(self.dir, r.data_file)
        _check(os.path.isfile(p), f"region {r.base:x}: region file {r.data_file} missing")
        return np.fromfile(p, dtype=np.uint8)

    def written_bytes(self, r: SnapRegion) -> np.ndarray:
        p = os.path.join(self.dir, "written", f"region_{self._hx(r)}.bin")
        if not r.written.size:
            _check(not os.path.exists(p) or os.path.getsize(p) == 0,
                   f"region {r.base:x}: written bytes present but W is empty")
            return np.zeros(0, dtype=np.uint8)
        _check(os.path.isfile(p), f"region {r.base:x}: written/region_{self._hx(r)}.bin missing")
        return np.fromfile(p, dtype=np.uint8)

    def post_state(self, r: SnapRegion) -> np.ndarray:
        """Post-dispatch bytes of a region.  POST: the region file.  PRE_W: the
        region file (pre-state) overlaid, chunk k of W at a time in ascending
        k, with the concatenated written bytes (R7)."""
        b = self.region_bytes(r).copy()
        if self.dispatch.get("mode") == "pre_w" and r.written.size:
            w = self.written_bytes(r)
            need = sum(min(CHUNK, r.size - int(k) * CHUNK) for k in r.written.tolist())
            _check(w.size == need, f"region {r.base:x}: written bytes {w.size} != {need} for |W|={r.written.size}")
            off = 0
            for k in r.written.tolist():
                lo = k * CHUNK
                ln = min(CHUNK, r.size - lo)
                b[lo:lo + ln] = w[off:off + ln]
                off += ln
        return b


def load(d: str) -> Snapshot:
    """Parse a kc-snapshot/1 directory.  Requires the sentinel (SPEC.md:412-426:
    a directory without ``capture_complete`` is an incomplete capture) and the
    three JSON files; the final per-region status is the one capture_log.json
    records (a region can fail after memory_regions.json was written first,
    PAPER.md:753-761)."""
    _check(os.path.isdir(d), f"{d}: not a directory")
    _check(os.path.exists(os.path.join(d, "capture_complete")), "no capture_complete sentinel")
    for f in ("dispatch.json", "memory_regions.json", "capture_log.json", "kernarg.bin"):
        _check(os.path.isfile(os.path.join(d, f)), f"{f} missing")
    with open(os.path.join(d, "dispatch.json")) as f:
        disp = json.load(f)
    with open(os.path.join(d, "memory_regions.json")) as f:
        mr = json.load(f)
    with open(os.path.join(d, "capture_log.json")) as f:
        log = json.load(f)
    _check(isinstance(mr, list), "memory_regions.json is not a list")
    _check(isinstance(log.get("regions"), list), "capture_log.json has no region list")
    logged = {}
    for e in log["regions"]:
        _check(e["base"] not in logged, f"capture_log.json lists region {e['base']} twice")
        logged[e["base"]] = e
    _check([e["base"] for e in log["regions"]] == [e["base"] for e in mr],
           "capture_log.json and memory_regions.json list different regions")
    regs = []
    for e in mr:
        hx = e["base"]
        _check(isinstance(hx, str) and _HEX_RE.match(hx) is not None, f"base {hx!r}: not lowercase hex without 0x")
        _check(_DIG_RE.match(e["digest"]) is not None, f"region {hx}: digest {e['digest']!r} is not 16 hex digits")
        le = logged[hx]
        _check(le["status"] in ("ok", "failed"), f"region {hx}: status {le['status']!r}")
        r = SnapRegion(int(hx, 16), int(e["size"]), e["alloc_kind"], le["status"], int(e["digest"], 16),
                       e["data_file"], n_chunks=int(e["n_chunks"]),
                       post_digest=int(le.get("post_digest", "0") or "0", 16),
                       logged_written=int(le.get("written_chunks", -1)))
        idx = os.path.join(d, "written", f"region_{hx}.idx")
        if os.path.exists(idx):
            r.written = _read_u64(idx, f"region {hx}: written index")
            r.has_idx = True
        regs.append(r)
    return Snapshot(d, disp, regs, log)


def cubin_module_vars(path: str) -> dict:
    """{name: size} of the user module variables of a CUDA ELF64 code object:
    STT_OBJECT symbols with a size, defined in a .nv.global* or .nv.constant*
    section other than the kernel parameter banks .nv.constant0.* (F3,
    PAPER.md:728-751).  Plain struct parsing of the ELF64 layout."""
    import struct
    b = open(path, "rb").read()
    assert b[:4] == b"\x7fELF" and b[4] == 2, "not an ELF64 code object"
    shoff, = struct.unpack_from("<Q", b, 0x28)
    shentsize, shnum, shstrndx = struct.unpack_from("<HHH", b, 0x3A)
    secs = [struct.unpack_from("<IIQQQQIIQQ", b, shoff + i * shentsize) for i in range(shnum)]
    # (name, type, flags, addr, offset, size, link, info, addralign, entsize)

    def cstr(off):
        return b[off:b.index(b"\0", off)].decode()
    shstr = secs[shstrndx]
    names = [cstr(shstr[4] + s[0]) for s in secs]
    out = {}
    for s in secs:
        if s[1] != 2:  # SHT_SYMTAB
            continue
        strtab = secs[s[6]]
        for o in range(0, s[5], s[9]):
            st_name, st_info, _, st_shndx, _, st_size = struct.unpack_from("<IBBHQQ", b, s[4] + o)
            if st_info & 0xF != 1 or st_size == 0 or st_shndx == 0 or st_shndx >= shnum:
                continue
            sec = names[st_shndx]
            if sec.startswith(".nv.global") or (sec.startswith(".nv.constant") and not sec.startswith(".nv.constant0")):
                out[cstr(strtab[4] + st_name)] = st_size
    return out


def verify(snap: Snapshot) -> dict:
    """Recompute and check everything the format promises; returns a summary.

    Raises SnapshotError on the first violation.  What is checked (DESIGN.md
    section 3):

    * dispatch.json: format, mode, hash parameters; kernarg.bin length and the
      parameter layout; kernel.cubin length and SHA-256 (the code object's
      identity);
    * regions sorted by base, non-overlapping, non-empty (R25, R6), with
      ``n_chunks = ceil(size / 65536)`` and data_file ``memory/region_<hex>.bin``;
    * per ``ok`` region: the region file is exactly ``size`` bytes; its
      manifest equals the recomputed chunk hashes and its digest the logged
      one (O2); the post manifest equals the hashes of the post state and the
      logged post digest its digest; the written index is sorted, unique and
      in range, its count matches capture_log.json, and (PRE_W) W equals the
      brute-force set of chunks whose pre and post bytes differ (O3) with the
      written bytes exactly the W chunks' lengths; (POST) the post manifest is
      the region manifest and no written bytes are stored;
    * capture_log.json: the written total and the snapshot digest S over the
      ``ok`` regions only (O2, R19).
    """
    d = snap.dir
    disp = snap.dispatch
    _check(disp.get("format") == "kc-snapshot/1", f"format {disp.get('format')!r}")
    mode = disp.get("mode")
    _check(mode in ("pre_w", "post"), f"mode {mode!r}")
    _check(disp.get("hash") == {"algo": "xxh64", "seed": 0, "chunk_bytes": CHUNK}, "hash parameters (R1, R2)")
    ka = os.path.getsize(os.path.join(d, "kernarg.bin"))
    _check(ka == disp["kernarg_size"], f"kernarg.bin has {ka} bytes, dispatch.json says {disp['kernarg_size']}")
    lay = disp.get("kernarg_layout", [])
    for a, b in zip(lay, lay[1:]):
        _check(int(a["offset"]) + int(a["size"]) <= int(b["offset"]), "kernarg_layout overlaps or is unsorted")
    if lay and ka:
        _check(int(lay[-1]["offset"]) + int(lay[-1]["size"]) == ka, "kernarg_layout does not end at kernarg_size")
    cub = os.path.join(d, "kernel.cubin")
    sha = disp.get("code_object_sha256", "")
    if sha:   # the code object's identity
        _check(os.path.isfile(cub), "kernel.cubin missing but dispatch.json names its SHA-256")
        _check(hashlib.sha256(open(cub, "rb").read()).hexdigest() == sha, "kernel.cubin SHA-256 mismatch")
    if disp.get("code_object_bytes"):
        _check(os.path.isfile(cub) and os.path.getsize(cub) == disp["code_object_bytes"],
               "kernel.cubin length != code_object_bytes")
    bases = [r.base for r in snap.regions]
    _check(bases == sorted(bases), "regions not sorted by base (R25)")
    for a, b in zip(snap.regions, snap.regions[1:]):
        _check(a.base + a.size <= b.base, f"regions {a.base:x} and {b.base:x} overlap")
    ok_bases, ok_sizes, ok_digs = [], [], []
    n_written = 0
    for r in snap.regions:
        hx = f"{r.base:x}"
        _check(r.size > 0, f"region {hx}: size 0")
        _check(r.n_chunks == n_chunks(r.size), f"region {hx}: n_chunks {r.n_chunks} != ceil({r.size}/65536)")
        _check(r.data_file == f"memory/region_{hx}.bin", f"region {hx}: data_file {r.data_file!r}")
        if r.status != "ok":
            continue
        data = snap.region_bytes(r)
        _check(data.size == r.size, f"region {hx}: file has {data.size} bytes, expected {r.size}")
        h = chunk_hashes(data)
        man = _read_u64(os.path.join(d, "memory", f"region_{hx}.xxh64"), f"region {hx}: manifest")
        _check(man.size == h.size and np.array_equal(h, man), f"region {hx}: manifest mismatch")
        dg = region_digest(h)
        _check(dg == r.digest, f"region {hx}: digest mismatch")
        _check(r.has_idx, f"region {hx}: written/region_{hx}.idx missing")
        w = r.written.astype(np.uint64)
        _check(all(int(a) < int(b) for a, b in zip(w[:-1], w[1:])), f"region {hx}: written index not sorted/unique")
        _check(w.size == 0 or int(w[-1]) < r.n_chunks, f"region {hx}: written index out of range")
        _check(r.logged_written == w.size, f"region {hx}: capture_log written_chunks {r.logged_written} != |W| {w.size}")
        pm = _read_u64(os.path.join(d, "post", f"region_{hx}.xxh64"), f"region {hx}: post manifest")
        post = snap.post_state(r)
        ph = chunk_hashes(post)
        _check(pm.size == ph.size and np.array_equal(ph, pm), f"region {hx}: post manifest mismatch")
        _check(region_digest(ph) == r.post_digest, f"region {hx}: capture_log post_digest mismatch")
        if mode == "pre_w":
            # W = chunks whose pre/post bytes differ (O3), by brute-force compare
            w_true = [k for k in range(r.n_chunks)
                      if not np.array_equal(data[k * CHUNK:(k + 1) * CHUNK], post[k * CHUNK:(k + 1) * CHUNK])]
            _check(w_true == w.tolist(), f"region {hx}: W {w.tolist()} != chunks that differ {w_true}")
            # and W is exactly the chunks whose manifests differ (A4)
            _check([k for k in range(r.n_chunks) if h[k] != pm[k]] == w.tolist(),
                   f"region {hx}: W != chunks whose pre/post hashes differ")
        else:
            _check(np.array_equal(pm, man), f"region {hx}: POST snapshot's post manifest != region manifest")
            p = os.path.join(d, "written", f"region_{hx}.bin")
            _check(not os.path.exists(p) or os.path.getsize(p) == 0, f"region {hx}: POST snapshot stores written bytes")
        n_written += int(w.size)
        ok_bases.append(r.base)
        ok_sizes.append(r.size)
        ok_digs.append(dg)
    _check(int(snap.log.get("written_chunks", -1)) == n_written,
           f"capture_log written_chunks {snap.log.get('written_chunks')} != {n_written}")
    S = snapshot_digest(ok_bases, ok_sizes, ok_digs)
    _check(_DIG_RE.match(snap.log.get("snapshot_digest", "")) is not None, "capture_log snapshot_digest malformed")
    _check(S == int(snap.log["snapshot_digest"], 16), "snapshot digest mismatch")
    # F3 module variables: every recorded variable is one the code object declares, with
    # its declared size, and both value files hold exactly that many bytes
    n_mv = 0
    mvp = os.path.join(d, "module_vars.json")
    if os.path.exists(mvp):
        mv = json.load(open(mvp))
        _check(mv["format"] == "kc-module-vars/1", "module_vars format")
        declared = cubin_module_vars(cub)
        for v in mv["vars"]:
            _check(declared.get(v["name"]) == v["size"], f"module variable {v['name']}: not declared with that size")
            pre = open(os.path.join(d, v["pre"]), "rb").read()
            post = open(os.path.join(d, v["post"]), "rb").read()
            _check(len(pre) == len(post) == v["size"], f"module variable {v['name']}: value file length")
            _check(v["written"] == (pre != post), f"module variable {v['name']}: written flag")
            n_mv += 1
    return {"regions": len(snap.regions), "ok": len(ok_bases), "written_chunks": n_written, "snapshot_digest": S,
            "module_vars": n_mv}


# --------------------------------------------------------------------------- F4 sequences
DEP_RAW, DEP_WAW, DEP_WAR = 1, 2, 4


def _pointer_regions(snap: Snapshot) -> set:
    """Regions (indices) that a pointer-sized kernarg parameter points into (R33)."""
    ka = open(os.path.join(snap.dir, "kernarg.bin"), "rb").read()
    out = set()
    for p in snap.dispatch.get("kernarg_layout", []):
        off, sz = int(p["offset"]), int(p["size"])
        if sz != 8 or off + 8 > len(ka):
            continue
        v = int.from_bytes(ka[off:off + 8], "little")
        for i, r in enumerate(snap.regions):
            if r.status == "ok" and r.base <= v < r.base + r.size:
                out.add(i)
    return out


def sequence_deps(steps: list) -> list:
    """Dependency flags of step j on step i < j, from the step directories
    alone (R33): RAW = a pointer parameter of j lies in a region i wrote; WAW =
    W_i and W_j share a chunk; WAR = a pointer parameter of i lies in a region
    j wrote."""
    n = len(steps)
    ptrs = [_pointer_regions(s) for s in steps]
    wch = [{(i, int(k)) for i, r in enumerate(s.regions) for k in r.written.tolist()} for s in steps]
    wreg = [{i for i, _ in w} for w in wch]
    deps = [[0] * n for _ in range(n)]
    for j in range(n):
        for i in range(j):
            f = 0
            if ptrs[j] & wreg[i]:
                f |= DEP_RAW
            if wch[j] & wch[i]:
                f |= DEP_WAW
            if ptrs[i] & wreg[j]:
                f |= DEP_WAR
            deps[j][i] = f
    return deps


def verify_sequence(d: str) -> dict:
    """Check a kc-sequence/1 directory (include/kc.h kc_seq_save): sentinel,
    every step a valid kc-snapshot/1 (verify), the chain identity -- the state
    before step k+1 is the state after step k, region by region, byte for byte
    (the dispatches ran back to back) -- and the dependency matrix recomputed
    from the step files (R33)."""
    _check(os.path.exists(os.path.join(d, "sequence_complete")), "no sequence_complete sentinel")
    meta = json.load(open(os.path.join(d, "sequence.json")))
    _check(meta.get("format") == "kc-sequence/1" and meta["n"] == len(meta["steps"]), "sequence.json header")
    _check(meta["n"] >= 1, "empty sequence")
    steps = [load(os.path.join(d, s["dir"])) for s in meta["steps"]]
    sums = [verify(s) for s in steps]
    for k, (s, m) in enumerate(zip(steps, meta["steps"])):
        _check(s.dispatch["mangled_symbol"] == m["mangled_symbol"], f"step {k}: symbol != sequence.json")
        _check(sum(int(r.written.size) for r in s.regions) == m["written_chunks"],
               f"step {k}: written_chunks != sequence.json")
    for k in range(len(steps) - 1):
        a, b = steps[k], steps[k + 1]
        _check([(r.base, r.size) for r in a.regions] == [(r.base, r.size) for r in b.regions],
               f"step {k} -> {k + 1}: region tables differ")
        for ra, rb in zip(a.regions, b.regions):
            if ra.status != "ok":
                continue
            _check(rb.status == "ok", f"step {k} -> {k + 1}: region {ra.base:x} lost")
            _check(np.array_equal(a.post_state(ra), b.region_bytes(rb)),
                   f"step {k} -> {k + 1}: region {ra.base:x} after step {k} != before step {k + 1}")
    deps = sequence_deps(steps)
    _check(deps == meta["deps"], f"dependency matrix {meta['deps']} != recomputed {deps}")
    return {"n": len(steps), "deps": deps, "written_chunks": [s["written_chunks"] for s in sums]}
