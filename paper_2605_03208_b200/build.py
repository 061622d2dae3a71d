"""Build libkc.so (sm_100a) in-tree with nvcc, plus the fixture cubin.

    python -m paper_2605_03208_b200.build            # build if stale
    python -m paper_2605_03208_b200.build --force

The library is the product path: hand-written CUDA kernels + the C ABI of
include/kc.h.  Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo,
NO fast-math, -fmad=false (exact IEEE fp64 in K2; reading R17).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkc.so")
FIXTURE_SRC = os.path.join(ROOT, "synth", "kc_fixtures.cu")
FIXTURE_CUBIN = os.path.join(ROOT, "synth", "kc_fixtures.cubin")
# variant code objects for the replay-override tests: an unmodified recompile
# (different optimisation level) and a modified kernel (KC_VARIANT_DELTA=1)
FIXTURE_VARIANTS = {os.path.join(ROOT, "synth", "kc_fixtures_recompiled.cubin"): ["-O1"],
                    os.path.join(ROOT, "synth", "kc_fixtures_modified.cubin"): ["-O3", "-DKC_VARIANT_DELTA=1"]}
# F4 workload: one attention-forward code object per "autotune config" BLOCK_N
ATTN_SRC = os.path.join(ROOT, "synth", "kc_attn_fwd.cu")
ATTN_BLOCK_N = (32, 64, 128)
ATTN_CUBINS = {bn: os.path.join(ROOT, "synth", f"kc_attn_fwd_n{bn}.cubin") for bn in ATTN_BLOCK_N}
# a retuned variant with another launch shape (BLOCK_M = 32: grid x2, 128 threads), same numerics
ATTN_M32_CUBIN = os.path.join(ROOT, "synth", "kc_attn_fwd_m32n64.cubin")
SOURCES = ["kc_kernels.cu", "kc_runtime.cu", "kc_snapshot.cu", "kc_module.cu", "kc_sequence.cu", "kc_interpose.cu"]
HEADERS = ["kc_kernels.cuh", "kc_internal.h", "kc_json.h", "kc_snapshot_types.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(PKG, "libkc_checked.so")


def build_lib(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """One object per translation unit, compiled in parallel (objects under
    build/, rebuilt when their source or any header changed), then linked.
    checked=True builds libkc_checked.so with -DKC_CHECKS=1 (device bounds checks
    on the rings, queues and chunk lookups; loaded when KC_LIB=checked)."""
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "kc.h"), __file__]
    objdir = os.path.join(ROOT, "build", "kc_obj_checked" if checked else "kc_obj")
    LIB = LIB_CHECKED if checked else globals()["LIB"]
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    todo = [(s, o) for s, o in zip(SOURCES, objs) if force or _stale(o, [os.path.join(CSRC, s)] + hdrs)]
    if not todo and not _stale(LIB, objs):
        return LIB
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-O2"]
    if checked:
        flags.append("-DKC_CHECKS=1")
    if verbose:
        flags.insert(0, "-Xptxas=-v")

    def compile_one(so):
        src, obj = so
        tmp = obj + f".tmp{os.getpid()}"
        cmd = [NVCC, *flags, "-c", "-o", tmp, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd, cwd=CSRC)
        os.replace(tmp, obj)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, todo))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"], cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


def build_fixtures(force: bool = False) -> str:
    for out, flags in [(FIXTURE_CUBIN, ["-O3"])] + list(FIXTURE_VARIANTS.items()):
        if force or _stale(out, [FIXTURE_SRC]):
            tmp = out + f".tmp{os.getpid()}"
            subprocess.check_call([NVCC, "-cubin", *ARCH, *flags, "-lineinfo", "-o", tmp, FIXTURE_SRC])
            os.replace(tmp, out)
    for bn, out in list(ATTN_CUBINS.items()) + [("m32", ATTN_M32_CUBIN)]:
        if force or _stale(out, [ATTN_SRC]):
            tmp = out + f".tmp{os.getpid()}"
            flags = ["-DKC_ATTN_BLOCK_M=32", "-DKC_ATTN_BLOCK_N=64"] if bn == "m32" else [f"-DKC_ATTN_BLOCK_N={bn}"]
            subprocess.check_call([NVCC, "-cubin", *ARCH, "-O3", "-lineinfo", *flags, "-o", tmp, ATTN_SRC])
            os.replace(tmp, out)
    return FIXTURE_CUBIN


def build(force: bool = False, verbose: bool = False) -> None:
    build_lib(force, verbose)
    build_fixtures(force)


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv, checked=True))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
