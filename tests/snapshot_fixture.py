"""Hand-built kc-snapshot/1 and kc-sequence/1 directories -- TEST INFRASTRUCTURE.

Writes the format of DESIGN.md section 3 (the paper's capture directory,
PAPER.md:681-697 [sec. 4.2.1], PAPER.md:937-953 [fig. reproducer]; sentinel
last) from hand-chosen bytes, using only ``oracle/`` (XXH64,
chunk manifests, digests, written set) and numpy.  It never touches the
product path.  The O1 checker (oracle/snapshot.py) is pinned against these
directories (tests/test_oracle_snapshot.py): the valid ones must verify, and
every corruption ``CORRUPTIONS`` applies must raise.

``python tests/snapshot_fixture.py --golden`` (re)writes
tests/golden/snapshot_fixture.txt: the fixture's chunk hashes, region digests
and S as this script computes them with the oracle.  The test recomputes
every line with python-xxhash (an independent library), so the golden file
pins the oracle's digests of the fixture, not the other way round.
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import struct
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

CHUNK = 65536
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "snapshot_fixture.txt")

# a fake code object: the checker only hashes it (SHA-256 identity)
CUBIN = b"KCFIXTURE-CODE-OBJECT-" + bytes(range(256)) * 3
SYMBOL = "_Z10kc_fixturePKmPmj"


def _pattern(n: int, mul: int, add: int) -> np.ndarray:
    i = np.arange(n, dtype=np.uint64)
    return ((i * mul + add + (i >> 13)) & 0xFF).astype(np.uint8)   # no two chunks alike


def fixture_regions():
    """Three regions with hand-chosen pre/post bytes (ascending bases, gaps between):

    * A @ 0x7f0000000000, 3 chunks + 100 B (a short last chunk): pre = (31 i + 7 + i // 8192) mod 256;
      the dispatch writes one byte of chunk 1 and the very last byte (chunk 3, short);
    * B @ 0x7f0000200000, 4,096 B of zeros, untouched by the dispatch;
    * C @ 0x7f0000400000, 2 chunks of 0xAB; the dispatch zeroes chunk 0 and rewrites
      chunk 1 with the same bytes it held (no change, so not in W).
    """
    a_pre = _pattern(3 * CHUNK + 100, 31, 7)
    a_post = a_pre.copy()
    a_post[CHUNK + 5] ^= 0x5A
    a_post[-1] ^= 0x01
    b_pre = np.zeros(4096, dtype=np.uint8)
    c_pre = np.full(2 * CHUNK, 0xAB, dtype=np.uint8)
    c_post = c_pre.copy()
    c_post[:CHUNK] = 0
    return [
        {"base": 0x7F0000000000, "pre": a_pre, "post": a_post, "kind": "vmm"},
        {"base": 0x7F0000200000, "pre": b_pre, "post": b_pre.copy(), "kind": "mem_alloc"},
        {"base": 0x7F0000400000, "pre": c_pre, "post": c_post, "kind": "vmm"},
    ]


def kernarg_for(regions) -> tuple[bytes, list]:
    """Packed parameter buffer (R22): two pointers (A, C) and a u32 count."""
    ka = struct.pack("<QQI", regions[0]["base"], regions[2]["base"], 40960) + b"\0" * 4
    return ka[:20], [{"offset": 0, "size": 8}, {"offset": 8, "size": 8}, {"offset": 16, "size": 4}]


def _hx(base: int) -> str:
    return f"{base:x}"


def write_snapshot(d: str, regions, mode: str = "pre_w", failed=(), kernarg=None, layout=None,
                   symbol: str = SYMBOL, cubin: bytes = CUBIN) -> dict:
    """Write a complete kc-snapshot/1 directory; returns what was written
    (per-region manifests and digests, S).  ``failed``: bases whose final
    status is "failed" (their region file is still written in PRE_W, as when a
    buffer is freed after the dispatch; S excludes them)."""
    if os.path.exists(d):
        shutil.rmtree(d)
    for sub in ("memory", "post", "written"):
        os.makedirs(os.path.join(d, sub))
    if kernarg is None:
        kernarg, layout = kernarg_for(regions)
    disp = {
        "format": "kc-snapshot/1", "mode": mode, "mangled_symbol": symbol, "cooperative": False,
        "grid": [32, 1, 1], "block": [256, 1, 1], "cluster": [1, 1, 1], "shared_mem_bytes": 0,
        "kernarg_size": len(kernarg), "device_ordinal": 0, "compute_capability": "10.0",
        "code_object_bytes": len(cubin), "kernarg_layout": layout,
        "code_object_sha256": hashlib.sha256(cubin).hexdigest(),
        "hash": {"algo": "xxh64", "seed": 0, "chunk_bytes": CHUNK},
    }
    # metadata first
    with open(os.path.join(d, "dispatch.json"), "w") as f:
        json.dump(disp, f, indent=2)
    open(os.path.join(d, "kernarg.bin"), "wb").write(kernarg)
    open(os.path.join(d, "kernel.cubin"), "wb").write(cubin)
    mr, lg, out = [], [], {"regions": []}
    ok_b, ok_s, ok_d, w_total = [], [], [], 0
    for r in regions:
        hx = _hx(r["base"])
        size = r["pre"].size
        stored = r["pre"] if mode == "pre_w" else r["post"]
        h = oracle.chunk_hashes(stored)
        ph = oracle.chunk_hashes(r["post"])
        dig, pdig = oracle.region_digest(h), oracle.region_digest(ph)
        w = np.nonzero(oracle.written_set(r["pre"], r["post"]))[0].astype("<u8")
        ok = r["base"] not in failed
        mr.append({"base": hx, "size": size, "alloc_kind": r["kind"], "device": 0, "contains_kernarg": False,
                   "data_file": f"memory/region_{hx}.bin", "n_chunks": oracle.n_chunks(size),
                   "digest": f"{dig:016x}", "status": "ok", "seq": len(mr)})
        stored.tofile(os.path.join(d, "memory", f"region_{hx}.bin"))
        if ok:
            h.astype("<u8").tofile(os.path.join(d, "memory", f"region_{hx}.xxh64"))
            ph.astype("<u8").tofile(os.path.join(d, "post", f"region_{hx}.xxh64"))
            w.tofile(os.path.join(d, "written", f"region_{hx}.idx"))
            if mode == "pre_w" and w.size:
                np.concatenate([r["post"][k * CHUNK:(k + 1) * CHUNK] for k in w.tolist()]).tofile(
                    os.path.join(d, "written", f"region_{hx}.bin"))
            ok_b.append(r["base"])
            ok_s.append(size)
            ok_d.append(dig)
            w_total += int(w.size)
        lg.append({"base": hx, "status": "ok" if ok else "failed",
                   "error": "" if ok else "freed between dispatch completion and snapshot",
                   "post_digest": f"{pdig if ok else 0:016x}", "written_chunks": int(w.size) if ok else 0})
        out["regions"].append({"base": r["base"], "size": size, "hashes": h, "post_hashes": ph, "digest": dig,
                               "post_digest": pdig, "written": w, "ok": ok})
    with open(os.path.join(d, "memory_regions.json"), "w") as f:
        json.dump(mr, f, indent=2)
    S = oracle.snapshot_digest(ok_b, ok_s, ok_d)
    with open(os.path.join(d, "capture_log.json"), "w") as f:
        json.dump({"regions": lg, "sink": "files", "snapshot_digest": f"{S:016x}", "written_chunks": w_total}, f,
                  indent=2)
    open(os.path.join(d, "capture_complete"), "wb").close()   # sentinel LAST
    out["S"] = S
    out["written_chunks"] = w_total
    return out


def sequence_states():
    """Three consecutive states of the fixture regions: s0 -> (step 0) -> s1 -> (step 1) -> s2.
    Step 0 is the fixture's dispatch; step 1 writes chunk 2 of A (RAW on A, which step 0
    wrote; WAW none; it also points at B)."""
    regs = fixture_regions()
    s0 = [r["pre"] for r in regs]
    s1 = [r["post"] for r in regs]
    s2 = [x.copy() for x in s1]
    s2[0][2 * CHUNK:2 * CHUNK + 8] = 0x11
    return regs, [s0, s1, s2]


def write_sequence(d: str) -> dict:
    """A kc-sequence/1 directory of two PRE_W steps (kc_seq_save's layout)."""
    if os.path.exists(d):
        shutil.rmtree(d)
    os.makedirs(d)
    regs, states = sequence_states()
    steps, meta = [], []
    params = [
        (struct.pack("<QQI", regs[0]["base"], regs[2]["base"], 7) + b"\0" * 4)[:20],
        (struct.pack("<QQ", regs[0]["base"] + 64, regs[1]["base"])),
    ]
    layouts = [
        [{"offset": 0, "size": 8}, {"offset": 8, "size": 8}, {"offset": 16, "size": 4}],
        [{"offset": 0, "size": 8}, {"offset": 8, "size": 8}],
    ]
    syms = [SYMBOL, "_Z7kc_stepPmPKm"]
    for k in range(2):
        rk = [{"base": r["base"], "kind": r["kind"], "pre": states[k][i], "post": states[k + 1][i]}
              for i, r in enumerate(regs)]
        sub = f"step_{k:03d}"
        info = write_snapshot(os.path.join(d, sub), rk, "pre_w", kernarg=params[k], layout=layouts[k], symbol=syms[k])
        steps.append(info)
        meta.append({"dir": sub, "mangled_symbol": syms[k], "written_chunks": info["written_chunks"]})
    # step 1's first pointer lies in A, which step 0 wrote: RAW; step 0's pointers (A, C) lie
    # in no region step 1 wrote except A: WAR; W_0 = {A1, A3, C0}, W_1 = {A2}: no WAW
    deps = [[0, 0], [1 | 4, 0]]
    with open(os.path.join(d, "sequence.json"), "w") as f:
        json.dump({"format": "kc-sequence/1", "n": 2, "steps": meta, "deps": deps}, f, indent=2)
    open(os.path.join(d, "sequence_complete"), "wb").close()
    return {"steps": steps, "deps": deps}


# --------------------------------------------------------------------------- corruptions
def _flip(path: str, off: int, mask: int = 0x01):
    b = bytearray(open(path, "rb").read())
    b[off if off >= 0 else len(b) + off] ^= mask
    open(path, "wb").write(bytes(b))


def _edit_json(path: str, fn):
    j = json.load(open(path))
    fn(j)
    json.dump(j, open(path, "w"), indent=2)


A, B, C = "7f0000000000", "7f0000200000", "7f0000400000"


def _p(d, *parts):
    return os.path.join(d, *parts)


def _shift_w(d):
    # W off by one chunk: the index says chunk 2 where chunk 1 was written (bytes unchanged)
    idx = np.fromfile(_p(d, "written", f"region_{A}.idx"), dtype="<u8")
    idx[0] += 1
    idx.tofile(_p(d, "written", f"region_{A}.idx"))


def _add_unwritten_chunk(d):
    # W lists chunk 0 of A (unchanged by the dispatch) with its unchanged bytes
    idx = np.fromfile(_p(d, "written", f"region_{A}.idx"), dtype="<u8")
    wb = np.fromfile(_p(d, "written", f"region_{A}.bin"), dtype=np.uint8)
    pre = np.fromfile(_p(d, "memory", f"region_{A}.bin"), dtype=np.uint8)
    np.concatenate([[0], idx]).astype("<u8").tofile(_p(d, "written", f"region_{A}.idx"))
    np.concatenate([pre[:CHUNK], wb]).tofile(_p(d, "written", f"region_{A}.bin"))


def _overlap(d):
    def f(mr):
        mr[1]["size"] = 0x7F0000400000 - 0x7F0000200000 + 1   # B now runs into C
        mr[1]["n_chunks"] = oracle.n_chunks(mr[1]["size"])
    _edit_json(_p(d, "memory_regions.json"), f)


def _unsort(d):
    def f(mr):
        mr[0], mr[1] = mr[1], mr[0]
    _edit_json(_p(d, "memory_regions.json"), f)

    def g(lg):
        lg["regions"][0], lg["regions"][1] = lg["regions"][1], lg["regions"][0]
    _edit_json(_p(d, "capture_log.json"), g)


def _set_log(key, fn):
    def f(d):
        _edit_json(_p(d, "capture_log.json"), lambda j: j.__setitem__(key, fn(j[key])))
    return f


def _set_region_log(i, key, val):
    def f(d):
        _edit_json(_p(d, "capture_log.json"), lambda j: j["regions"][i].__setitem__(key, val))
    return f


def _set_mr(i, key, val):
    def f(d):
        _edit_json(_p(d, "memory_regions.json"), lambda j: j[i].__setitem__(key, val))
    return f


def _rm(*parts):
    def f(d):
        os.remove(_p(d, *parts))
    return f


def _truncate(*parts):
    def f(d):
        p = _p(d, *parts)
        b = open(p, "rb").read()
        open(p, "wb").write(b[:-1])
    return f


# name -> corruption of a valid PRE_W fixture; each must make verify (or load) raise
CORRUPTIONS = {
    "sentinel_missing": _rm("capture_complete"),
    "manifest_byte_flipped": lambda d: _flip(_p(d, "memory", f"region_{A}.xxh64"), 9),
    "post_manifest_byte_flipped": lambda d: _flip(_p(d, "post", f"region_{C}.xxh64"), 3),
    "region_byte_flipped": lambda d: _flip(_p(d, "memory", f"region_{B}.bin"), 100),
    "region_file_truncated": _truncate("memory", f"region_{A}.bin"),
    "region_file_missing": _rm("memory", f"region_{B}.bin"),
    "manifest_missing": _rm("memory", f"region_{B}.xxh64"),
    "post_manifest_missing": _rm("post", f"region_{A}.xxh64"),
    "written_idx_dropped": _rm("written", f"region_{A}.idx"),
    "written_idx_dropped_empty_w": _rm("written", f"region_{B}.idx"),
    "written_bin_dropped": _rm("written", f"region_{C}.bin"),
    "written_bin_truncated": _truncate("written", f"region_{A}.bin"),
    "written_byte_flipped": lambda d: _flip(_p(d, "written", f"region_{A}.bin"), 5),
    "w_off_by_one_chunk": _shift_w,
    "w_extra_unchanged_chunk": _add_unwritten_chunk,
    "sha256_mismatch": lambda d: _flip(_p(d, "kernel.cubin"), 40),
    "cubin_missing": _rm("kernel.cubin"),
    "kernarg_truncated": _truncate("kernarg.bin"),
    "overlapping_regions": _overlap,
    "unsorted_regions": _unsort,
    "snapshot_digest_wrong": _set_log("snapshot_digest", lambda s: f"{int(s, 16) ^ 1:016x}"),
    "written_total_wrong": _set_log("written_chunks", lambda n: n + 1),
    "post_digest_wrong": _set_region_log(2, "post_digest", "0123456789abcdef"),
    "region_written_count_wrong": _set_region_log(0, "written_chunks", 1),
    "region_digest_wrong": _set_mr(1, "digest", "0000000000000001"),
    "n_chunks_wrong": _set_mr(0, "n_chunks", 3),
    "data_file_renamed": _set_mr(0, "data_file", "memory/other.bin"),
    "base_uppercase_hex": _set_mr(0, "base", A.upper()),
    "log_region_missing": lambda d: _edit_json(_p(d, "capture_log.json"), lambda j: j["regions"].pop(1)),
    "mode_unknown": lambda d: _edit_json(_p(d, "dispatch.json"), lambda j: j.__setitem__("mode", "pre")),
    "hash_chunk_changed": lambda d: _edit_json(_p(d, "dispatch.json"),
                                               lambda j: j["hash"].__setitem__("chunk_bytes", 4096)),
}


def _break_chain(d):
    # the state before step 1 is no longer the state after step 0 (one byte of B)
    p = _p(d, "step_001", "memory", f"region_{B}.bin")
    _flip(p, 7)
    # keep step 1 internally consistent so only the chain identity can catch it
    pre = np.fromfile(p, dtype=np.uint8)
    h = oracle.chunk_hashes(pre)
    h.astype("<u8").tofile(_p(d, "step_001", "memory", f"region_{B}.xxh64"))
    h.astype("<u8").tofile(_p(d, "step_001", "post", f"region_{B}.xxh64"))
    dg = oracle.region_digest(h)
    _edit_json(_p(d, "step_001", "memory_regions.json"), lambda j: j[1].__setitem__("digest", f"{dg:016x}"))
    _edit_json(_p(d, "step_001", "capture_log.json"), lambda j: j["regions"][1].__setitem__("post_digest", f"{dg:016x}"))
    mr = json.load(open(_p(d, "step_001", "memory_regions.json")))
    S = oracle.snapshot_digest([int(e["base"], 16) for e in mr], [e["size"] for e in mr],
                               [int(e["digest"], 16) for e in mr])
    _edit_json(_p(d, "step_001", "capture_log.json"), lambda j: j.__setitem__("snapshot_digest", f"{S:016x}"))


SEQ_CORRUPTIONS = {
    "sequence_sentinel_missing": _rm("sequence_complete"),
    "broken_chain_identity": _break_chain,
    "deps_wrong": lambda d: _edit_json(_p(d, "sequence.json"), lambda j: j.__setitem__("deps", [[0, 0], [1, 0]])),
    "step_count_wrong": lambda d: _edit_json(_p(d, "sequence.json"),
                                             lambda j: j["steps"][1].__setitem__("written_chunks", 9)),
    "step_invalid": lambda d: _flip(_p(d, "step_000", "memory", f"region_{A}.xxh64"), 0),
}


def golden_lines() -> list[str]:
    """One line per value the golden file pins: chunk hashes, region digests, S."""
    info = write_snapshot("/tmp/_kc_fixture_golden", fixture_regions(), "pre_w")
    shutil.rmtree("/tmp/_kc_fixture_golden")
    lines = []
    for r in info["regions"]:
        for k, h in enumerate(r["hashes"].tolist()):
            lines.append(f"chunk {r['base']:x} {k} {h:016x}")
        for k, h in enumerate(r["post_hashes"].tolist()):
            lines.append(f"post_chunk {r['base']:x} {k} {h:016x}")
        lines.append(f"digest {r['base']:x} {r['digest']:016x}")
        lines.append(f"post_digest {r['base']:x} {r['post_digest']:016x}")
        lines.append(f"written {r['base']:x} {' '.join(str(int(k)) for k in r['written'].tolist()) or '-'}")
    lines.append(f"S {info['S']:016x}")
    return lines


if __name__ == "__main__":
    if "--golden" in sys.argv:
        with open(GOLDEN, "w") as f:
            f.write("# kc-snapshot/1 fixture (tests/snapshot_fixture.py fixture_regions, PRE_W) as computed by\n"
                    "# `python tests/snapshot_fixture.py --golden` with oracle/ only.  Every hash is re-derived\n"
                    "# with python-xxhash in tests/test_oracle_snapshot.py (O2: XXH64 seed 0 per 64 KiB chunk,\n"
                    "# region digest over LE64 chunk hashes, S over LE64 base|size|digest by ascending base).\n")
            f.write("\n".join(golden_lines()) + "\n")
        print("wrote", GOLDEN)
    else:
        d = sys.argv[1] if len(sys.argv) > 1 else "/tmp/kc_fixture"
        print(json.dumps({"S": write_snapshot(d, fixture_regions())["S"]}))
