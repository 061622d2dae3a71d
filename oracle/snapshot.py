"""O1: independent reader/checker of the kc-snapshot/1 directory -- TEST INFRASTRUCTURE.

Parses the capture directory with Python's json (not the product's C++
parser), checks every file's length, recomputes every manifest and digest
with the oracle's own XXH64 (oracle/kc_oracle.c) and checks the sentinel
(DESIGN.md "Snapshot
format").  Never imports the product path.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import CHUNK, chunk_hashes, n_chunks, region_digest, snapshot_digest


@dataclass
class SnapRegion:
    base: int
    size: int
    kind: str
    status: str
    digest: int
    data_file: str
    written: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))


@dataclass
class Snapshot:
    dir: str
    dispatch: dict
    regions: list
    log: dict

    def region_bytes(self, r: SnapRegion) -> np.ndarray:
        return np.fromfile(os.path.join(self.dir, r.data_file), dtype=np.uint8)

    def written_bytes(self, r: SnapRegion) -> np.ndarray:
        p = os.path.join(self.dir, "written", f"region_{r.base:x}.bin")
        return np.fromfile(p, dtype=np.uint8) if os.path.exists(p) else np.zeros(0, dtype=np.uint8)

    def post_state(self, r: SnapRegion) -> np.ndarray:
        """Post-dispatch bytes of a region: PRE_W = region file overlaid with written chunks."""
        b = self.region_bytes(r).copy()
        if self.dispatch.get("mode") == "pre_w" and r.written.size:
            w = self.written_bytes(r)
            off = 0
            for k in r.written.tolist():
                lo = k * CHUNK
                ln = min(CHUNK, r.size - lo)
                b[lo:lo + ln] = w[off:off + ln]
                off += ln
        return b


def load(d: str) -> Snapshot:
    if not os.path.exists(os.path.join(d, "capture_complete")):
        raise ValueError("no capture_complete sentinel")
    with open(os.path.join(d, "dispatch.json")) as f:
        disp = json.load(f)
    with open(os.path.join(d, "memory_regions.json")) as f:
        mr = json.load(f)
    with open(os.path.join(d, "capture_log.json")) as f:
        log = json.load(f)
    final = {e["base"]: e["status"] for e in log["regions"]}
    regs = []
    for e in mr:
        r = SnapRegion(int(e["base"], 16), int(e["size"]), e["alloc_kind"], final.get(e["base"], e["status"]),
                       int(e["digest"], 16), e["data_file"])
        idx = os.path.join(d, "written", f"region_{e['base']}.idx")
        if os.path.exists(idx):
            r.written = np.fromfile(idx, dtype="<u8")
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

    Raises AssertionError on the first violation."""
    d = snap.dir
    assert snap.dispatch["format"] == "kc-snapshot/1"
    assert snap.dispatch["hash"] == {"algo": "xxh64", "seed": 0, "chunk_bytes": CHUNK}
    bases = [r.base for r in snap.regions]
    assert bases == sorted(bases), "regions not sorted by base (R25)"
    for a, b in zip(snap.regions, snap.regions[1:]):
        assert a.base + a.size <= b.base, "regions overlap"
    ka = os.path.getsize(os.path.join(d, "kernarg.bin"))
    assert ka == snap.dispatch["kernarg_size"]
    cub = os.path.join(d, "kernel.cubin")
    if snap.dispatch.get("code_object_bytes"):
        assert os.path.getsize(cub) == snap.dispatch["code_object_bytes"]
    if snap.dispatch.get("code_object_sha256"):   # the code object's identity
        import hashlib
        assert hashlib.sha256(open(cub, "rb").read()).hexdigest() == snap.dispatch["code_object_sha256"]
    ok_bases, ok_sizes, ok_digs = [], [], []
    n_written = 0
    for r in snap.regions:
        if r.status != "ok":
            continue
        data = snap.region_bytes(r)
        assert data.size == r.size, f"region {r.base:x}: file has {data.size} bytes, expected {r.size}"
        h = chunk_hashes(data)
        man = np.fromfile(os.path.join(d, "memory", f"region_{r.base:x}.xxh64"), dtype="<u8")
        assert np.array_equal(h, man), f"region {r.base:x}: manifest mismatch"
        dg = region_digest(h)
        assert dg == r.digest, f"region {r.base:x}: digest mismatch"
        post = snap.post_state(r)
        ph = chunk_hashes(post)
        pm_path = os.path.join(d, "post", f"region_{r.base:x}.xxh64")
        if os.path.exists(pm_path):
            assert np.array_equal(ph, np.fromfile(pm_path, dtype="<u8")), f"region {r.base:x}: post manifest"
        if snap.dispatch.get("mode") == "pre_w":
            wexp = sum(min(CHUNK, r.size - k * CHUNK) for k in r.written.tolist())
            assert snap.written_bytes(r).size == wexp
            # W = chunks whose pre/post bytes differ (O3)
            pre = data
            w_true = [k for k in range(n_chunks(r.size))
                      if not np.array_equal(pre[k * CHUNK:(k + 1) * CHUNK], post[k * CHUNK:(k + 1) * CHUNK])]
            assert w_true == sorted(r.written.tolist())
        n_written += int(r.written.size)
        ok_bases.append(r.base)
        ok_sizes.append(r.size)
        ok_digs.append(dg)
    S = snapshot_digest(ok_bases, ok_sizes, ok_digs)
    logged = int(snap.log["snapshot_digest"], 16)
    assert S == logged, "snapshot digest mismatch"
    # F3 module variables: every recorded variable is one the code object declares, with
    # its declared size, and both value files hold exactly that many bytes
    n_mv = 0
    mvp = os.path.join(d, "module_vars.json")
    if os.path.exists(mvp):
        mv = json.load(open(mvp))
        assert mv["format"] == "kc-module-vars/1"
        declared = cubin_module_vars(cub)
        for v in mv["vars"]:
            assert declared.get(v["name"]) == v["size"], f"module variable {v['name']}: not declared with that size"
            pre = open(os.path.join(d, v["pre"]), "rb").read()
            post = open(os.path.join(d, v["post"]), "rb").read()
            assert len(pre) == len(post) == v["size"]
            assert v["written"] == (pre != post)
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
    from the step files."""
    assert os.path.exists(os.path.join(d, "sequence_complete")), "no sequence_complete sentinel"
    meta = json.load(open(os.path.join(d, "sequence.json")))
    assert meta["format"] == "kc-sequence/1" and meta["n"] == len(meta["steps"])
    steps = [load(os.path.join(d, s["dir"])) for s in meta["steps"]]
    sums = [verify(s) for s in steps]
    for k, (s, m) in enumerate(zip(steps, meta["steps"])):
        assert s.dispatch["mangled_symbol"] == m["mangled_symbol"]
        assert sum(int(r.written.size) for r in s.regions) == m["written_chunks"]
    for k in range(len(steps) - 1):
        a, b = steps[k], steps[k + 1]
        assert [(r.base, r.size) for r in a.regions] == [(r.base, r.size) for r in b.regions]
        for ra, rb in zip(a.regions, b.regions):
            if ra.status != "ok":
                continue
            assert np.array_equal(a.post_state(ra), b.region_bytes(rb)), \
                f"step {k} -> {k + 1}: region {ra.base:x} after step {k} != before step {k + 1}"
    deps = sequence_deps(steps)
    assert deps == meta["deps"], f"dependency matrix {meta['deps']} != recomputed {deps}"
    return {"n": len(steps), "deps": deps, "written_chunks": [s["written_chunks"] for s in sums]}
