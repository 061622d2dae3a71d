"""Subprocess worker for the closure tests (capture in one process, restore /
replay / validate in a fresh one).  Prints one JSON line on stdout.

    python tests/closure_worker.py capture-c1 DIR --mode pre_w|post [--mutate] [--free REGION]
    python tests/closure_worker.py capture-c2 DIR
    python tests/closure_worker.py replay DIR [--iterations N] [--no-recopy] [--squat]
    python tests/closure_worker.py recapture DIR OUT2     # restore then snapshot again (round trip)
"""
import argparse
import json
import time
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2605_03208_b200 import kc  # noqa: E402


def _upload(va, arr):
    import torch
    v = synth.dev_view(va, arr.size)
    v.copy_(torch.from_numpy(np.ascontiguousarray(arr)))
    torch.cuda.synchronize()


def _download(va, n):
    import torch
    v = synth.dev_view(va, n)
    return v.cpu().numpy()


def capture_c1(a):
    ctx = kc.Context(0, io_chunk_bytes=a.io_chunk)
    sizes = [s.size for s in synth.C1_SPECS]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va = vas
    nodes, heads, out = synth.c1_fill(nodes_va)
    for va, arr in zip(vas, (nodes, heads, out)):
        _upload(va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    karg = synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=int(a.mutate))
    if a.free:
        os.environ["KC_TEST_FREE_AFTER_DISPATCH"] = f"{vas[a.free]:x}"
    mode = kc.KC_MODE_PRE_W if a.mode == "pre_w" else kc.KC_MODE_POST
    rc, rep = ctx.capture(a.dir, image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                          kernarg=karg, mode=mode)
    # the original dispatch's post-state (what the replay must reproduce)
    if not a.free:
        np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_orig_out.npy"), _download(out_va, sizes[2]))
        np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_orig_nodes.npy"), _download(nodes_va, sizes[0]))
    print(json.dumps({"rc": rc, "report": rep, "vas": vas}))


def capture_c2(a):
    import torch
    ctx = kc.Context(0)
    specs = synth.c2_specs()
    gen = torch.Generator(device="cuda").manual_seed(synth.seed(2))
    va = {}
    for s in specs:
        p = ctx.alloc(s.size)
        va[s.name] = p
        synth.fill_device(synth.dev_view(p, s.size), s, gen)
    torch.cuda.synchronize()
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    rc, rep = ctx.capture(a.dir, image=image, mangled="kc_fixture_decode_attn", grid=(32, 1, 1), block=(128, 1, 1),
                          kernarg=synth.c2_kernarg(va), mode=kc.KC_MODE_PRE_W)
    np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_orig_out.npy"),
            _download(va["attn_out"], specs[[s.name for s in specs].index("attn_out")].size))
    print(json.dumps({"rc": rc, "report": rep, "vas": va}))


def _windows(d):
    with open(os.path.join(d, "memory_regions.json")) as f:
        regs = json.load(f)
    W = 32 << 20
    out = []
    for r in sorted(regs, key=lambda r: int(r["base"], 16)):
        lo = int(r["base"], 16) // W * W
        hi = (int(r["base"], 16) + int(r["size"]) + W - 1) // W * W
        if out and lo <= out[-1][1]:
            out[-1][1] = max(out[-1][1], hi)
        else:
            out.append([lo, hi])
    return out


def squat(a):
    """Occupy every captured VA window with a host PROT_NONE mapping (after CUDA
    initialises: a mapping present at cuInit is excluded from the driver's VA
    space for good, R28): restore must abort with
    KC_ERR_VA_UNAVAILABLE and leave nothing behind; once the squatter unmaps,
    the same restore must succeed."""
    import ctypes
    libc = ctypes.CDLL(None, use_errno=True)
    libc.mmap.restype = ctypes.c_void_p
    libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
    libc.munmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    flags = 0x02 | 0x20 | 0x4000 | 0x100000  # PRIVATE | ANONYMOUS | NORESERVE | FIXED_NOREPLACE
    attempt = int(os.environ.get("KC_REEXEC_ATTEMPT", "0"))

    def again(why):
        if attempt < 8:
            os.environ["KC_REEXEC_ATTEMPT"] = str(attempt + 1)
            os.execv(sys.executable, [sys.executable] + sys.argv)
        return {"error": why}

    ctx = kc.Context(0)
    held = []
    for lo, hi in _windows(a.dir):
        p = libc.mmap(lo, hi - lo, 0, flags, -1, 0)
        if p != lo:
            for l2, h2 in held:
                libc.munmap(l2, h2 - l2)
            return again("window occupied before the squat")
        held.append((lo, hi))
    out = {"squat": [0, held[0][0], held[0][0]], "attempts": attempt + 1}
    try:
        r0, _ = ctx.restore(a.dir)
        out["restore"] = "unexpected success"
        r0.release()
    except kc.KcError as e:
        out["restore_status"] = e.status
        out["message"] = str(e)
    out["squat_free"] = sum(int(libc.munmap(lo, hi - lo)) for lo, hi in held)
    # the aborted restore left nothing behind and the ctx is healthy: hash a fresh buffer
    p = ctx.alloc(1 << 20)
    import torch
    h = torch.zeros(16, dtype=torch.int64, device="cuda")
    ctx.hash([(p, 1 << 20)], h.data_ptr())
    torch.cuda.synchronize()
    ctx.free(p)
    out["ctx_healthy_after_abort"] = True
    return out


def replay(a):
    if a.squat:
        print(json.dumps(squat(a)))
        return
    if not a.no_prereserve:  # stage 2: claim the captured VA windows before CUDA initialises
        kc.exec_replay_process(sys.argv, a.dir)
    ctx = kc.Context(0)
    out = {"attempts": int(os.environ.get("KC_REEXEC_ATTEMPT", "0")) + 1}
    try:
        r, rep = kc.restore_in_fresh_layout(ctx, a.dir, sys.argv)
    except kc.KcError as e:
        print(json.dumps({"restore_status": e.status, "message": str(e), "report": getattr(e, "report", None)}))
        return
    out["restore"] = rep
    out["regions"] = [[x.base, x.size] for x in r.regions()]
    dump = os.path.join(a.dir, "..", os.path.basename(a.dir) + "_replay")
    override = open(a.override, "rb").read() if a.override else None
    out["replay"] = ctx.replay(r, iterations=a.iterations, no_recopy=a.no_recopy, dump_dir=dump,
                               image_override=override)
    if a.typed:  # typed validation of one output range: "<hex va>:<nbytes>:<dtype>"
        va, nb, dt = a.typed.split(":")
        treps, _ = ctx.validate(r, outs=[(int(va, 16), int(nb), dt)])
        out["typed"] = treps
    reps, unexpected = ctx.validate(r)
    out["validate"] = reps
    out["unexpected_chunks"] = unexpected
    out["modvars"] = ctx.validate_module_vars(r)
    out["dump"] = dump
    r.release()
    print(json.dumps(out))


def recapture(a):
    kc.exec_replay_process(sys.argv, a.dir)
    ctx = kc.Context(0)
    r, rep = kc.restore_in_fresh_layout(ctx, a.dir, sys.argv)
    regs = r.regions()
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    # a no-op dispatch (zero lists): the snapshot must equal the restored state
    karg = synth.c1_kernarg(0, 0, 0, n_lists=0)
    rc, rep2 = ctx.capture(a.out, image=image, mangled="kc_fixture_walk", grid=(1, 1, 1), block=(32, 1, 1),
                           kernarg=karg, regions=[(x.base, x.size) for x in regs], mode=kc.KC_MODE_PRE_W)
    r.release()
    print(json.dumps({"rc": rc, "restore": rep, "capture": rep2}))


def inproc(a):
    """Capture c1 from cuMemAlloc'd regions, free them, restore in the same
    process (cuMemAlloc replay for driver-pooled VA), replay, validate."""
    ctx = kc.Context(0, alloc_mode=kc.KC_ALLOC_MEMALLOC if a.memalloc else kc.KC_ALLOC_VMM)
    sizes = [s.size for s in synth.C1_SPECS]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va = vas
    for va, arr in zip(vas, synth.c1_fill(nodes_va)):
        _upload(va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    rc, rep = ctx.capture(a.dir, image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                          kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=1))
    orig = _download(out_va, sizes[2])
    for va in vas:
        ctx.free(va)
    out = {"rc": rc, "vas": vas}
    try:
        r, rrep = ctx.restore(a.dir)
    except kc.KcError as e:
        out.update({"restore_status": e.status, "message": str(e)})
        print(json.dumps(out))
        return
    out["restore"] = rrep
    out["replay"] = ctx.replay(r)
    reps, unexpected = ctx.validate(r)
    out["validate"] = reps
    out["unexpected_chunks"] = unexpected
    out["out_equal"] = bool(np.array_equal(_download(out_va, sizes[2]), orig))
    r.release()
    print(json.dumps(out))


def devsnap(a):
    """F1: capture c1 into a device arena, persist it (for the oracle), free the
    live regions, restore from the arena at the same VAs, replay, validate."""
    ctx = kc.Context(0)
    sizes = [s.size for s in synth.C1_SPECS]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va = vas
    for va, arr in zip(vas, synth.c1_fill(nodes_va)):
        _upload(va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    mode = kc.KC_MODE_PRE_W if a.mode == "pre_w" else kc.KC_MODE_POST
    snap, rep = ctx.capture_dev(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                                kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=int(a.mutate)),
                                mode=mode, host=a.host)
    orig_out = _download(out_va, sizes[2])
    np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_orig_out.npy"), orig_out)
    snap.save(a.dir)
    out = {"capture": rep, "vas": vas, "arena_bytes": snap.nbytes(), "is_host": snap.is_host()}
    for va in vas:
        ctx.free(va)
    # restore -> replay -> validate -> release, `cycles` times in this process:
    # every cycle must land on the captured VAs (the ctx VA heap, R28d)
    out["cycles"] = []
    for c in range(a.cycles):
        r, rrep = ctx.restore_dev(snap)
        cyc = {"restore": rrep, "regions": [[x.base, x.size] for x in r.regions()], "replay": ctx.replay(r),
               "out_equal": bool(np.array_equal(_download(out_va, sizes[2]), orig_out))}
        cyc["typed"], _ = ctx.validate(r, outs=[(out_va, sizes[2], "u64")])
        cyc["validate"], cyc["unexpected_chunks"] = ctx.validate(r)
        r.release()
        out["cycles"].append(cyc)
    out.update(out["cycles"][0])
    snap.free()
    print(json.dumps(out))


def devsnap_inplace(a):
    """kc_restore_dev_into: restore c1 once (kc_restore_dev), then `cycles` times capture
    from the restored state and restore the new snapshot over the live restore (no VA or
    physical operations); every replay must reproduce the output its capture observed, and
    a snapshot of other regions is refused."""
    ctx = kc.Context(0)
    sizes = [s.size for s in synth.C1_SPECS]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va = vas
    for va, arr in zip(vas, synth.c1_fill(nodes_va)):
        _upload(va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    disp = dict(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=int(a.mutate)), mode=kc.KC_MODE_PRE_W,
                regions=sorted(zip(vas, sizes)))
    snap, rep = ctx.capture_dev(**disp)
    for va in vas:
        ctx.free(va)
    r, rrep = ctx.restore_dev(snap)
    snap.free()
    out = {"cycles": []}
    for c in range(a.cycles):
        _upload(out_va, np.zeros(sizes[2], dtype=np.uint8))  # a fresh output buffer: W != {}
        snap, rep = ctx.capture_dev(**disp)
        seen = _download(out_va, sizes[2])
        rrep = ctx.restore_dev_into(snap, r)
        after_restore = _download(out_va, sizes[2])
        cyc = {"capture": rep, "restore": rrep, "regions": [[x.base, x.size] for x in r.regions()],
               "restored_pre": bool(np.array_equal(after_restore, np.zeros(sizes[2], dtype=np.uint8))),
               "replay": ctx.replay(r)}
        cyc["out_equal"] = bool(np.array_equal(_download(out_va, sizes[2]), seen))
        cyc["validate"], cyc["unexpected_chunks"] = ctx.validate(r)
        out["cycles"].append(cyc)
        snap.free()
    # a snapshot of other regions is refused
    other = ctx.alloc(65536)
    _upload(other, np.ones(65536, dtype=np.uint8))
    snap_o, _ = ctx.capture_dev(image=image, mangled="kc_fixture_walk", grid=(1, 1, 1), block=(32, 1, 1),
                                kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=0),
                                mode=kc.KC_MODE_PRE_W, regions=[(other, 65536)])
    try:
        ctx.restore_dev_into(snap_o, r)
        out["refused"] = False
    except kc.KcError as e:
        out["refused"] = e.status == kc.KC_ERR_ARG
    snap_o.free()
    r.release()
    out["vas"] = vas
    print(json.dumps(out))


def incr(a):
    """F2 incremental capture: a full capture, then one against it (only the
    chunks the first dispatch wrote are copied), the base freed, the second
    persisted for the oracle and restored/replayed/validated."""
    ctx = kc.Context(0)
    sizes = [s.size for s in synth.C1_SPECS]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va = vas
    for va, arr in zip(vas, synth.c1_fill(nodes_va)):
        _upload(va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    disp = dict(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=0), mode=kc.KC_MODE_PRE_W, host=a.host)
    snap0, rep0 = ctx.capture_dev(**disp)
    orig_out = _download(out_va, sizes[2])
    # the second dispatch also mutates the nodes (its W is the 10 node chunks)
    disp["kernarg"] = synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=1)
    snap1, rep1 = ctx.capture_dev(base=snap0, **disp)
    out = {"rep0": rep0, "rep1": rep1, "bytes0": snap0.nbytes(), "bytes1": snap1.nbytes(),
           "shared1": snap1.shared_bytes(), "sizes": sizes, "vas": vas}
    snap0.free()  # snap1 keeps the base bytes it references
    snap1.save(a.dir)
    for va in vas:
        ctx.free(va)
    r, rrep = ctx.restore_dev(snap1)
    out["restore"] = rrep
    out["replay"] = ctx.replay(r)
    out["out_equal"] = bool(np.array_equal(_download(out_va, sizes[2]), orig_out))
    out["validate"], out["unexpected_chunks"] = ctx.validate(r)
    out["typed"], _ = ctx.validate(r, outs=[(nodes_va, sizes[0], "u32")])
    r.release()
    snap1.free()
    print(json.dumps(out))


def capture_modvar(a):
    """F3: the application loads the fixture module itself (cuda-python), sets
    its __constant__ / __device__ variables, and the capture gets only the
    CUfunction (+ the image unless the CUPTI hook recorded the module load)."""
    import struct
    from cuda.bindings import driver as drv
    ctx = kc.Context(0)
    if a.cupti:
        ctx.track_install()
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    err, mod = drv.cuModuleLoadData(image)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    err, fn = drv.cuModuleGetFunction(mod, b"kc_fixture_modvar")
    assert err == drv.CUresult.CUDA_SUCCESS, err

    def put(name, arr):
        err, p, sz = drv.cuModuleGetGlobal(mod, name)
        assert err == drv.CUresult.CUDA_SUCCESS and sz == arr.nbytes, (err, sz)
        drv.cuMemcpyHtoD(p, arr.ctypes.data, arr.nbytes)
    put(b"kc_fixture_cvals", (np.arange(1, 9, dtype=np.uint32) * 7))
    put(b"kc_fixture_scale", np.array([3.25], dtype=np.float32))
    put(b"kc_fixture_hits", np.array([1000], dtype=np.uint64))
    n = 5000
    out_va = ctx.alloc(8 * n)
    _upload(out_va, np.zeros(n, dtype=np.uint64))
    karg = struct.pack("<QI", out_va, n)
    rc, rep = ctx.capture(a.dir, func=int(fn), image=None if a.cupti else image, grid=((n + 255) // 256, 1, 1),
                          block=(256, 1, 1), kernarg=karg, mode=kc.KC_MODE_PRE_W)
    np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_orig_out.npy"), _download(out_va, 8 * n))
    print(json.dumps({"rc": rc, "report": rep, "out_va": out_va, "n": n}))


def publish(a):
    """F1 across processes: capture c1 into a device arena, persist a normal copy
    for the oracle (<dir>_files), publish the arena (CUDA IPC) to <dir>, and
    replay it in a fresh process while this one keeps the snapshot alive."""
    import subprocess
    ctx = kc.Context(0)
    sizes = [s.size for s in synth.C1_SPECS]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va = vas
    for va, arr in zip(vas, synth.c1_fill(nodes_va)):
        _upload(va, arr)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    disp = dict(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=int(a.mutate)), mode=kc.KC_MODE_PRE_W)
    snap, rep = ctx.capture_dev(**disp)
    out = {"capture": rep, "vas": vas}
    snap.save(a.dir + "_files")
    snap.publish(a.dir)
    # refused: a host snapshot and an incremental one (bytes not in one own arena)
    hs, _ = ctx.capture_host(**disp)
    inc, _ = ctx.capture_dev(base=snap, **disp)
    out["refused"] = []
    for s_ in (hs, inc):
        try:
            s_.publish(a.dir + "_refused")
            out["refused"].append(0)
        except kc.KcError as e:
            out["refused"].append(e.status)
        s_.free()
    p = subprocess.run([sys.executable, __file__, "replay", a.dir], capture_output=True, text=True, timeout=300)
    out["child_rc"] = p.returncode
    out["child"] = json.loads(p.stdout.strip().splitlines()[-1]) if p.stdout.strip() else {"stderr": p.stderr[-2000:]}
    snap.free()
    # the publisher's arena is gone: a late replay must fail cleanly
    p = subprocess.run([sys.executable, __file__, "replay", a.dir, "--no-prereserve"], capture_output=True, text=True,
                       timeout=300)
    out["late"] = json.loads(p.stdout.strip().splitlines()[-1]) if p.stdout.strip() else {"stderr": p.stderr[-2000:]}
    print(json.dumps(out))


def interpose(a):
    """A3 interposed mode: an application drives the CUDA driver API itself
    (module load, cuMemAlloc, two launches of the list walk); the library only
    installs its CUPTI hook and arms the capture of launch #1 (the in-place
    F1' walk).  Reports the capture status and what the application saw."""
    import ctypes
    import struct
    from cuda.bindings import driver as drv
    ctx = kc.Context(0)
    ctx.track_install()
    target_dir = "/proc/kc_not_writable/cap" if a.bad_dir else a.dir   # a capture that must fail
    ctx.interpose_arm("kc_fixture_walk", 1, target_dir, kc.KC_MODE_POST if a.mode == "post" else kc.KC_MODE_PRE_W)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    err, mod = drv.cuModuleLoadData(image)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    err, fn = drv.cuModuleGetFunction(mod, b"kc_fixture_walk")
    sizes = [s.size for s in synth.C1_SPECS]
    ptrs = []
    for sz in sizes:
        err, p_ = drv.cuMemAlloc(sz)
        assert err == drv.CUresult.CUDA_SUCCESS, err
        ptrs.append(int(p_))
    nodes, heads, out = ptrs
    init = synth.c1_fill(nodes)
    for p_, arr in zip(ptrs, init):
        drv.cuMemcpyHtoD(p_, arr.ctypes.data, arr.nbytes)
    types = (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int)
    for mutate in (0, 1):   # launch #0 (not captured), launch #1 (captured, rewrites the nodes)
        args = ((heads, out, nodes, synth.C1_N_LISTS, mutate), types)
        err, = drv.cuLaunchKernel(fn, 32, 1, 1, 256, 1, 1, 0, 0, args, 0)
        assert err == drv.CUresult.CUDA_SUCCESS, err
    drv.cuCtxSynchronize()
    st = ctx.interpose_status()
    got = []
    for p_, sz in zip(ptrs, sizes):
        h = np.zeros(sz, dtype=np.uint8)
        drv.cuMemcpyDtoH(h.ctypes.data, p_, sz)
        got.append(h)
    os.makedirs(a.dir, exist_ok=True)   # (a failed capture never created it)
    np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_app_nodes.npy"), got[0])
    np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_app_out.npy"), got[2])
    np.save(os.path.join(a.dir, "..", os.path.basename(a.dir) + "_init_nodes.npy"), init[0])
    print(json.dumps({"status": st, "ptrs": ptrs, "tracked": [[r.base, r.size] for r in ctx.regions()]}))


def interpose_seq(a):
    """F4 from an unmodified application: the library arms a 3-launch sequence
    capture; the application (driver API) runs walk(mutate=1), axpy, walk."""
    import ctypes
    from cuda.bindings import driver as drv
    ctx = kc.Context(0)
    ctx.track_install()
    ctx.interpose_arm_seq(None, 0, 3)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    err, mod = drv.cuModuleLoadData(image)
    err, walk = drv.cuModuleGetFunction(mod, b"kc_fixture_walk")
    err, axpy = drv.cuModuleGetFunction(mod, b"kc_fixture_axpy_u32")
    n_y = 100_003
    sizes = [s.size for s in synth.C1_SPECS] + [4 * n_y, 4 * n_y]
    ptrs = []
    for sz in sizes:
        err, p_ = drv.cuMemAlloc(sz)
        ptrs.append(int(p_))
    nodes, heads, out, x, y = ptrs
    rng = np.random.default_rng(5)
    init = list(synth.c1_fill(nodes)) + [rng.integers(0, 2**32, n_y, dtype=np.uint64).astype(np.uint32),
                                         rng.integers(0, 2**32, n_y, dtype=np.uint64).astype(np.uint32)]
    for p_, arr in zip(ptrs, init):
        drv.cuMemcpyHtoD(p_, arr.ctypes.data, arr.nbytes)
    wt = (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int)
    drv.cuLaunchKernel(walk, 32, 1, 1, 256, 1, 1, 0, 0, ((heads, out, nodes, synth.C1_N_LISTS, 1), wt), 0)
    drv.cuLaunchKernel(axpy, (n_y + 255) // 256, 1, 1, 256, 1, 1, 0, 0,
                       ((x, y, n_y, 7), (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32)), 0)
    drv.cuLaunchKernel(walk, 32, 1, 1, 256, 1, 1, 0, 0, ((heads, out, nodes, synth.C1_N_LISTS, 0), wt), 0)
    drv.cuCtxSynchronize()
    st = ctx.interpose_status()
    seq = ctx.interpose_take_seq()
    deps = seq.deps()
    seq.save(a.dir)
    seq.free()
    print(json.dumps({"status": st, "deps": deps, "ptrs": ptrs}))


def load_replay(a):
    """Capture once, replay many: a fresh process loads a
    file snapshot into HBM once (kc_snapshot_load), then restores at the
    captured VAs, replays and validates `cycles` times from memory."""
    if not a.no_prereserve:
        kc.exec_replay_process(sys.argv, a.dir)
    ctx = kc.Context(0)
    t0 = time.perf_counter()
    snap = ctx.load_snapshot(a.dir, host=a.host)
    out = {"load_s": time.perf_counter() - t0, "is_host": snap.is_host(), "cycles": []}
    for _ in range(a.cycles):
        t1 = time.perf_counter()
        try:
            r, rst = ctx.restore_dev(snap)
        except kc.KcError as e:   # the driver's arenas landed on a captured VA: fresh layout (R28c)
            if e.status == kc.KC_ERR_VA_UNAVAILABLE:
                kc._reexec(sys.argv, 8)
            raise
        t2 = time.perf_counter()
        ctx.replay(r)
        reps, unexpected = ctx.validate(r)
        t3 = time.perf_counter()
        out["cycles"].append({"restore_s": t2 - t1, "replay_validate_s": t3 - t2, "verify": rst["verify_mismatch_chunks"],
                              "regions": [[x.base, x.size] for x in r.regions()],
                              "ok": all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0 and len(reps) > 0})
        r.release()
    snap.free()
    print(json.dumps(out))


def load_seq(a):
    """A saved sequence loaded in a fresh process and replayed jointly."""
    # every step covers the same regions: the pre-CUDA collision check of step 0
    # (re-exec for a fresh ASLR layout, R28c) protects the whole joint replay
    kc.exec_replay_process(sys.argv, os.path.join(a.dir, "step_000"))
    ctx = kc.Context(0)
    seq = ctx.load_seq(a.dir)
    steps, _ = kc.replay_seq_in_fresh_layout(ctx, seq, sys.argv)
    out = {"n": len(seq), "deps": seq.deps(), "steps": steps}
    seq.free()
    print(json.dumps(out))


def interpose_graph(a):
    """A launch recorded by stream capture (CUDA graph) is not a dispatch that runs:
    the hook skips it; the graph replays, then the direct launch is captured."""
    import ctypes
    from cuda.bindings import driver as drv
    ctx = kc.Context(0)
    ctx.track_install()
    ctx.interpose_arm("kc_fixture_walk", 0, a.dir, kc.KC_MODE_PRE_W)
    err, mod = drv.cuModuleLoadData(open(synth.FIXTURE_CUBIN, "rb").read())
    err, fn = drv.cuModuleGetFunction(mod, b"kc_fixture_walk")
    sizes = [s.size for s in synth.C1_SPECS]
    ptrs = [int(drv.cuMemAlloc(sz)[1]) for sz in sizes]
    nodes, heads, out = ptrs
    init = synth.c1_fill(nodes)
    for p_, arr in zip(ptrs, init):
        drv.cuMemcpyHtoD(p_, arr.ctypes.data, arr.nbytes)
    err, stream = drv.cuStreamCreate(0)
    types = (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int)
    drv.cuStreamBeginCapture(stream, drv.CUstreamCaptureMode.CU_STREAM_CAPTURE_MODE_RELAXED)
    drv.cuLaunchKernel(fn, 32, 1, 1, 256, 1, 1, 0, stream, ((heads, out, nodes, synth.C1_N_LISTS, 0), types), 0)
    err, graph = drv.cuStreamEndCapture(stream)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    err, gexec = drv.cuGraphInstantiate(graph, 0)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    seen_after_capture = ctx.interpose_status()["seen"]
    drv.cuGraphLaunch(gexec, stream)
    drv.cuStreamSynchronize(stream)
    drv.cuLaunchKernel(fn, 32, 1, 1, 256, 1, 1, 0, stream, ((heads, out, nodes, synth.C1_N_LISTS, 1), types), 0)
    drv.cuStreamSynchronize(stream)
    st = ctx.interpose_status()
    h = np.zeros(sizes[0], dtype=np.uint8)
    drv.cuMemcpyDtoH(h.ctypes.data, nodes, sizes[0])
    dt = np.dtype([("next", "<u8"), ("value", "<u4"), ("pad", "<u4")])
    v0 = init[0].view(dt)["value"].astype(np.uint64)
    once = bool(np.array_equal(h.view(dt)["value"], ((3 * v0 + 1) % 2**32).astype(np.uint32)))
    print(json.dumps({"status": st, "seen_after_capture": seen_after_capture, "mutated_once": once}))


def capture_gap(a):
    """Two regions less than one 32 MiB VA window apart, the second starting
    inside the first one's window and ending past it (the restore's
    window merge).  A: 2 MiB at w + 2 MiB, B: 8 MiB at w + 28 MiB (w 32 MiB
    aligned); the pad and the 24 MiB filler between them are freed before
    the capture."""
    M = 1 << 20
    ctx = kc.Context(0)
    probe = ctx.alloc(2 * M)
    ctx.free(probe)
    pad_sz = ((2 * M - probe) % (32 * M)) or 32 * M
    pad = ctx.alloc(pad_sz)
    A = ctx.alloc(2 * M)
    filler = ctx.alloc(24 * M)
    B = ctx.alloc(8 * M)
    ctx.free(filler)
    ctx.free(pad)
    geom = {"A": A, "B": B, "a_off": A % (32 * M), "b_off": B - A // (32 * M) * (32 * M)}
    rng = np.random.default_rng(7)
    _upload(A, rng.integers(0, 256, 2 * M, dtype=np.uint8))
    _upload(B, rng.integers(0, 256, 8 * M, dtype=np.uint8))
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    rc, rep = ctx.capture(a.dir, image=image, mangled="kc_fixture_walk", grid=(1, 1, 1), block=(32, 1, 1),
                          kernarg=synth.c1_kernarg(0, 0, 0, n_lists=0), regions=[(A, 2 * M), (B, 8 * M)],
                          mode=kc.KC_MODE_PRE_W)
    print(json.dumps({"rc": rc, "geom": geom, "report": rep}))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("cmd")
    p.add_argument("dir")
    p.add_argument("out", nargs="?")
    p.add_argument("--mode", default="pre_w")
    p.add_argument("--mutate", action="store_true")
    p.add_argument("--free", type=int, default=0)
    p.add_argument("--io-chunk", type=int, default=0)
    p.add_argument("--iterations", type=int, default=1)
    p.add_argument("--no-recopy", action="store_true")
    p.add_argument("--squat", action="store_true")
    p.add_argument("--no-prereserve", action="store_true")
    p.add_argument("--memalloc", action="store_true")
    p.add_argument("--override", default=None)
    p.add_argument("--typed", default=None)
    p.add_argument("--host", action="store_true")
    p.add_argument("--cycles", type=int, default=1)
    p.add_argument("--cupti", action="store_true")
    p.add_argument("--bad-dir", action="store_true")
    a = p.parse_args()
    {"capture-c1": capture_c1, "capture-c2": capture_c2, "replay": replay, "recapture": recapture,
     "inproc": inproc, "devsnap": devsnap, "devsnap-inplace": devsnap_inplace, "incr": incr, "capture-modvar": capture_modvar,
     "publish": publish, "interpose": interpose, "interpose-seq": interpose_seq, "load-replay": load_replay,
     "load-seq": load_seq, "interpose-graph": interpose_graph,
     "capture-gap": capture_gap}[a.cmd](a)


if __name__ == "__main__":
    main()
