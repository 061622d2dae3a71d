"""kc command line: the paper's capture / replay workflow (PAPER.md:141-151,
1061-1135) over libkc.so.

    python -m paper_2605_03208_b200.cli capture --kernel NAME [--index N] [--mode pre_w|post] --out DIR -- CMD ...
    python -m paper_2605_03208_b200.cli replay DIR [--override CUBIN [--grid X,Y,Z --block X,Y,Z --smem B
                                                  --symbol NAME]] [--iterations N] [--no-recopy] [--dump]
                                                  [--typed HEXVA:NBYTES:DTYPE] [--atol A --rtol R]
    python -m paper_2605_03208_b200.cli capture --kernel NAME --index N --count K --out DIR -- CMD ...   (a sequence)
    python -m paper_2605_03208_b200.cli replay-seq DIR
    python -m paper_2605_03208_b200.cli info DIR

`capture` runs an unmodified CUDA application with CUDA_INJECTION64_PATH
pointing at libkc.so: the driver loads the library at cuInit
(InitializeInjection), its CUPTI hook tracks the application's allocations and
module loads, and brackets launch number N of the first kernel whose name
contains NAME (A3 interposed mode).  The application must use the device's
primary context (the CUDA runtime, PyTorch and Triton do).  `replay` restores
the snapshot at the captured VAs in this (fresh) process, replays the dispatch
(optionally a variant code object, the paper's --hsaco) and validates it; one
JSON report on stdout.  Argument marshalling only: the work is in libkc.so.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

# absolute imports: a replay re-execs this file as a script for a fresh VA layout
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _capture(a, rest) -> int:
    from paper_2605_03208_b200 import kc
    if not rest:
        print("capture: missing the application command after --", file=sys.stderr)
        return 2
    env = dict(os.environ, CUDA_INJECTION64_PATH=kc.LIB_PATH, KC_CAPTURE_DIR=os.path.abspath(a.out),
               KC_TARGET=a.kernel or "", KC_DISPATCH_INDEX=str(a.index), KC_CAPTURE_MODE=a.mode,
               KC_CAPTURE_COUNT=str(a.count))
    p = subprocess.run(rest, env=env)
    done = os.path.exists(os.path.join(a.out, "capture_complete" if a.count <= 1 else "sequence_complete"))
    print(json.dumps({"app_returncode": p.returncode, "captured": done, "dir": os.path.abspath(a.out)}))
    return 0 if done else 1


def _replay(a) -> int:
    from paper_2605_03208_b200 import kc
    kc.exec_replay_process(sys.argv, a.dir)      # pre-CUDA VA collision check (re-exec for a fresh layout)
    ctx = kc.Context(0)
    r, rst = kc.restore_in_fresh_layout(ctx, a.dir, sys.argv)
    override = open(a.override, "rb").read() if a.override else None
    dump = os.path.abspath(a.dir.rstrip("/") + "_replay") if a.dump else None
    shape = lambda v: tuple(int(x) for x in v.split(",")) if v else None  # noqa: E731
    rep = ctx.replay(r, iterations=a.iterations, no_recopy=a.no_recopy, dump_dir=dump, image_override=override,
                     grid=shape(a.grid), block=shape(a.block), smem=a.smem, symbol=a.symbol)
    out = {"restore": rst, "replay": rep, "process_layouts": int(os.environ.get("KC_REEXEC_ATTEMPT", "0")) + 1}
    if a.typed:
        va, nb, dt = a.typed.split(":")
        out["typed"], _ = ctx.validate(r, outs=[(int(va, 16), int(nb), dt)], atol=a.atol, rtol=a.rtol)
    out["validate"], out["unexpected_chunks"] = ctx.validate(r, atol=a.atol, rtol=a.rtol)
    out["module_vars"] = ctx.validate_module_vars(r)
    out["pass"] = (all(x["pass"] == 1 for x in out["validate"]) and out["unexpected_chunks"] == 0
                   and all(x["pass"] == 1 for x in out.get("typed", [])))
    if dump:
        out["dump"] = dump
    r.release()
    ctx.close()
    print(json.dumps(out))
    return 0 if out["pass"] else 3


def _replay_seq(a) -> int:
    from paper_2605_03208_b200 import kc
    kc.exec_replay_process(sys.argv, os.path.join(a.dir, "step_000"))  # every step has the same regions
    ctx = kc.Context(0)
    seq = ctx.load_seq(a.dir)
    steps, _ = kc.replay_seq_in_fresh_layout(ctx, seq, sys.argv, atol=a.atol, rtol=a.rtol)
    out = {"n": len(seq), "deps": seq.deps(), "steps": steps, "pass": all(s["pass"] == 1 for s in steps)}
    seq.free()
    ctx.close()
    print(json.dumps(out))
    return 0 if out["pass"] else 3


def _info(a) -> int:
    d = a.dir
    disp = json.load(open(os.path.join(d, "dispatch.json")))
    regs = json.load(open(os.path.join(d, "memory_regions.json")))
    log = json.load(open(os.path.join(d, "capture_log.json")))
    print(json.dumps({"kernel": disp.get("mangled_symbol"), "grid": disp.get("grid"), "block": disp.get("block"),
                      "mode": disp.get("mode"), "code_object_sha256": disp.get("code_object_sha256"),
                      "regions": len(regs), "bytes": sum(int(r["size"]) for r in regs),
                      "written_chunks": log.get("written_chunks"),
                      "snapshot_digest": log.get("snapshot_digest"),
                      "device_resident": os.path.exists(os.path.join(d, "memory", "device_arena.json"))}))
    return 0


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    rest = []
    if "--" in argv:
        i = argv.index("--")
        argv, rest = argv[:i], argv[i + 1:]
    p = argparse.ArgumentParser(prog="kc")
    sub = p.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("capture")
    c.add_argument("--kernel", default="")
    c.add_argument("--index", type=int, default=0)
    c.add_argument("--mode", default="pre_w", choices=["pre_w", "post"])
    c.add_argument("--out", required=True)
    c.add_argument("--count", type=int, default=1, help="consecutive launches to capture as a sequence (F4)")
    r = sub.add_parser("replay")
    r.add_argument("dir")
    r.add_argument("--override", default=None)
    r.add_argument("--iterations", type=int, default=1)
    r.add_argument("--no-recopy", action="store_true")
    r.add_argument("--grid", default=None, help="launch-shape override for a retuned variant, e.g. 128,32")
    r.add_argument("--block", default=None, help="e.g. 128")
    r.add_argument("--smem", type=int, default=None, help="dynamic shared memory bytes")
    r.add_argument("--symbol", default=None, help="kernel name in the override code object")
    r.add_argument("--dump", action="store_true")
    r.add_argument("--typed", default=None)
    r.add_argument("--atol", type=float, default=1e-8)
    r.add_argument("--rtol", type=float, default=1e-5)
    q = sub.add_parser("replay-seq")
    q.add_argument("dir")
    q.add_argument("--atol", type=float, default=1e-8)
    q.add_argument("--rtol", type=float, default=1e-5)
    i_ = sub.add_parser("info")
    i_.add_argument("dir")
    a = p.parse_args(argv)
    if a.cmd == "capture":
        return _capture(a, rest)
    if a.cmd == "replay":
        return _replay(a)
    if a.cmd == "replay-seq":
        return _replay_seq(a)
    return _info(a)


if __name__ == "__main__":
    sys.exit(main())
