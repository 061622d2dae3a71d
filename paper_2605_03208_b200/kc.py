"""Thin ctypes binding of libkc.so (include/kc.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels and C++ runtime;
this module only converts Python values to the C ABI and back.  There is no
fallback: if libkc.so is missing or does not load, :func:`lib` raises.

Device memory is passed as integer device virtual addresses (e.g.
``torch.Tensor.data_ptr()`` or :meth:`Context.alloc`), streams as integer
CUstream handles (``torch.cuda.current_stream().cuda_stream``; 0 = default).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Iterable, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
# KC_LIB=checked loads the bounds-checked build (libkc_checked.so, -DKC_CHECKS=1)
LIB_PATH = os.path.join(_PKG, "libkc_checked.so" if os.environ.get("KC_LIB") == "checked" else "libkc.so")

KC_CHUNK_BYTES = 65536

# kc_status
KC_OK, KC_PARTIAL = 0, 1
KC_ERR_ARG, KC_ERR_STATE, KC_ERR_CUDA, KC_ERR_IO, KC_ERR_FORMAT = -1, -2, -3, -4, -5
KC_ERR_VA_UNAVAILABLE, KC_ERR_NOT_TRACKED, KC_ERR_OUT_OF_BOUNDS, KC_ERR_NOMEM = -6, -7, -8, -9
KC_ERR_MANIFEST_MISMATCH, KC_ERR_UNSUPPORTED = -10, -11
# kc_event / kc_alloc_kind / kc_capture_mode
KC_EV_ALLOC, KC_EV_FREE, KC_EV_MAP, KC_EV_UNMAP = 0, 1, 2, 3
KC_KIND_MEMALLOC, KC_KIND_VMM, KC_KIND_POOL = 0, 1, 2
KC_MODE_PRE_W, KC_MODE_POST = 0, 1
KC_ALLOC_VMM, KC_ALLOC_MEMALLOC = 0, 1
# kc_dtype
DTYPES = ["bytes", "u8", "i8", "u16", "i16", "u32", "i32", "u64", "i64", "f16", "bf16", "f32", "f64"]
DT = {n: i for i, n in enumerate(DTYPES)}
ELEM_SIZE = [1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8]

EXPORTED = [
    "kc_create", "kc_destroy", "kc_last_error", "kc_abi_version", "kc_build_info", "kc_status_str",
    "kc_kernel_launches", "kc_track",
    "kc_regions", "kc_alloc", "kc_free", "kc_track_install", "kc_track_uninstall", "kc_hash", "kc_count_chunks",
    "kc_hash_plan_create", "kc_hash_plan_run", "kc_hash_plan_chunks", "kc_hash_plan_destroy",
    "kc_diff_plan_create", "kc_diff_plan_run", "kc_diff_plan_destroy",
    "kc_written", "kc_diff_async", "kc_hash_diff_async", "kc_diff", "kc_capture", "kc_restore", "kc_prereserve", "kc_replay",
    "kc_validate", "kc_restored_regions", "kc_release", "kc_capture_dev", "kc_restore_dev", "kc_restore_dev_into",
    "kc_snapshot_save",
    "kc_snapshot_bytes", "kc_snapshot_free", "kc_capture_host", "kc_host_arena_reserve", "kc_snapshot_is_host",
    "kc_capture_incr", "kc_snapshot_shared_bytes", "kc_validate_module_vars",
    "kc_snapshot_publish", "kc_dev_arena_reserve", "kc_validate_host_ref",
    "kc_interpose_arm", "kc_interpose_status", "kc_interpose_take", "kc_interpose_arm_seq", "kc_interpose_take_seq",
    "kc_snapshot_load", "kc_seq_load", "kc_capture_seq", "kc_seq_length", "kc_seq_step", "kc_seq_deps", "kc_seq_save", "kc_seq_free", "kc_replay_seq",
    "kc_report_finalize", "kc_peer_export", "kc_peer_import", "kc_peer_release",
]
KC_DEP_RAW, KC_DEP_WAW, KC_DEP_WAR = 1, 2, 4


class KcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{status_name(status)}: {msg}")
        self.status = status


# ----------------------------------------------------------------- ABI structs
class Region(ctypes.Structure):
    _fields_ = [("base", ctypes.c_uint64), ("size", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("seq", ctypes.c_uint64)]

    def __repr__(self):
        return f"Region(base=0x{self.base:x}, size={self.size}, device={self.device}, kind={self.kind})"


class Buffer(ctypes.Structure):
    _fields_ = [("ref", ctypes.c_uint64), ("act", ctypes.c_uint64), ("nbytes", ctypes.c_uint64),
                ("dtype", ctypes.c_int32), ("report", ctypes.c_int32), ("bitmap_chunk0", ctypes.c_uint64)]


class Tolerance(ctypes.Structure):
    _fields_ = [("atol", ctypes.c_double), ("rtol", ctypes.c_double), ("equal_nan", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


class DiffReport(ctypes.Structure):
    _fields_ = [
        ("nbytes", ctypes.c_uint64), ("n_elems", ctypes.c_uint64), ("n_chunks", ctypes.c_uint64),
        ("differing_bytes", ctypes.c_uint64), ("differing_elems", ctypes.c_uint64), ("max_ulp", ctypes.c_uint64),
        ("max_abs", ctypes.c_double), ("max_rel", ctypes.c_double), ("percent_bytes", ctypes.c_double),
        ("nan_ref", ctypes.c_uint64), ("nan_act", ctypes.c_uint64), ("nan_pos_mismatch", ctypes.c_uint64),
        ("rel_undefined", ctypes.c_uint64), ("allclose_fail", ctypes.c_uint64),
        ("pass_", ctypes.c_int32), ("_pad", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {n: getattr(self, n) for n, _ in self._fields_ if n != "_pad"}
        d["pass"] = d.pop("pass_")
        return d


class Dispatch(ctypes.Structure):
    _fields_ = [("func", ctypes.c_void_p), ("image", ctypes.c_void_p), ("image_size", ctypes.c_size_t),
                ("mangled", ctypes.c_char_p), ("grid", ctypes.c_uint32 * 3), ("block", ctypes.c_uint32 * 3),
                ("smem_bytes", ctypes.c_uint32), ("kernarg_size", ctypes.c_uint32), ("kernarg", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("cluster", ctypes.c_uint32 * 3), ("flags", ctypes.c_uint32)]


class Options(ctypes.Structure):
    _fields_ = [("io_chunk_bytes", ctypes.c_uint64), ("pinned_depth", ctypes.c_uint32), ("device", ctypes.c_int32),
                ("alloc_mode", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class CaptureReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "n_regions", "n_chunks", "total_bytes", "n_failed_regions", "written_chunks", "d2h_bytes", "dma_calls",
        "staging_high_water", "snapshot_digest")] + [(n, ctypes.c_double) for n in (
            "t_hash_pre_s", "t_d2h_s", "t_dispatch_s", "t_hash_post_s", "t_total_s")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class ReplayOpts(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint32), ("no_recopy", ctypes.c_int32), ("dump_dir", ctypes.c_char_p),
                ("image_override", ctypes.c_void_p), ("image_override_size", ctypes.c_size_t),
                ("stream", ctypes.c_void_p), ("overrides", ctypes.c_uint32), ("grid", ctypes.c_uint32 * 3),
                ("block", ctypes.c_uint32 * 3), ("smem_bytes", ctypes.c_uint32), ("symbol", ctypes.c_char_p)]


class ReplayReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint32), ("module_vars_restored", ctypes.c_uint32),
                ("kernel_ms_mean", ctypes.c_double),
                ("kernel_ms_min", ctypes.c_double), ("kernel_ms_max", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "_pad"}


class RestoreReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "n_regions", "n_spans", "mapped_bytes", "h2d_bytes", "n_failed_regions", "verify_mismatch_chunks")] + [
        (n, ctypes.c_double) for n in ("t_reserve_s", "t_h2d_s", "t_verify_s", "t_total_s")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class SeqReplayOpts(ctypes.Structure):
    _fields_ = [("first", ctypes.c_size_t), ("count", ctypes.c_size_t),
                ("image_overrides", ctypes.POINTER(ctypes.c_void_p)), ("image_override_sizes", ctypes.POINTER(ctypes.c_size_t)),
                ("tol", Tolerance), ("stream", ctypes.c_void_p)]


class SeqStepReport(ctypes.Structure):
    _fields_ = [("w", DiffReport), ("unexpected_chunks", ctypes.c_uint64), ("inherited_chunks", ctypes.c_uint64),
                ("modvar_mismatch", ctypes.c_uint64), ("kernel_ms", ctypes.c_double), ("pass_", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]

    def as_dict(self) -> dict:
        return {"w": self.w.as_dict(), "unexpected_chunks": self.unexpected_chunks,
                "inherited_chunks": self.inherited_chunks,
                "modvar_mismatch": self.modvar_mismatch, "kernel_ms": self.kernel_ms, "pass": self.pass_}


# ----------------------------------------------------------------- loading
_lib = None


def lib() -> ctypes.CDLL:
    """Load libkc.so (built in-tree by ``python -m paper_2605_03208_b200.build``).

    Raises if it is missing: the product path has no CPU or Python fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2605_03208_b200.build` "
                          "(there is no fallback for the CUDA path)")
    L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_LOCAL)
    P, V, U64, I32, SZ = ctypes.POINTER, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_size_t
    st = ctypes.c_int
    sig = {
        "kc_create": (st, [P(V), P(Options)]),
        "kc_destroy": (None, [V]),
        "kc_last_error": (ctypes.c_char_p, [V]),
        "kc_abi_version": (ctypes.c_int, []),
        "kc_build_info": (ctypes.c_char_p, []),
        "kc_status_str": (ctypes.c_char_p, [st]),
        "kc_kernel_launches": (U64, [V]),
        "kc_track": (st, [V, ctypes.c_int, U64, U64, I32, I32]),
        "kc_regions": (st, [V, P(Region), SZ, P(SZ)]),
        "kc_alloc": (st, [V, U64, P(U64)]),
        "kc_free": (st, [V, U64]),
        "kc_track_install": (st, [V]),
        "kc_track_uninstall": (st, [V]),
        "kc_hash": (st, [V, P(Region), SZ, V, V, V, V]),
        "kc_count_chunks": (U64, [P(Region), SZ]),
        "kc_written": (st, [V, V, V, U64, V, V, V]),
        "kc_diff_async": (st, [V, P(Buffer), SZ, SZ, P(U64), P(U64), P(Tolerance), V, V, V]),
        "kc_hash_diff_async": (st, [V, P(Buffer), SZ, P(Tolerance), V, V, V, V, V]),
        "kc_diff": (st, [V, P(Buffer), SZ, P(Tolerance), P(DiffReport), P(U64), V]),
        "kc_validate_host_ref": (st, [V, P(Buffer), SZ, V, P(Tolerance), P(DiffReport), P(U64), V, P(U64), V]),
        "kc_capture": (st, [V, P(Dispatch), P(Region), SZ, ctypes.c_char_p, ctypes.c_int, P(CaptureReport)]),
        "kc_restore": (st, [V, ctypes.c_char_p, P(V), P(RestoreReport)]),
        "kc_prereserve": (st, [ctypes.c_char_p, P(U64)]),
        "kc_replay": (st, [V, V, P(ReplayOpts), P(ReplayReport)]),
        "kc_validate": (st, [V, V, P(Buffer), SZ, P(Tolerance), P(DiffReport), SZ, P(SZ), P(U64)]),
        "kc_restored_regions": (st, [V, P(Region), SZ, P(SZ)]),
        "kc_release": (None, [V]),
        "kc_capture_dev": (st, [V, P(Dispatch), P(Region), SZ, ctypes.c_int, P(V), P(CaptureReport)]),
        "kc_restore_dev": (st, [V, V, P(V), P(RestoreReport)]),
        "kc_restore_dev_into": (st, [V, V, V, P(RestoreReport)]),
        "kc_snapshot_save": (st, [V, V, ctypes.c_char_p]),
        "kc_snapshot_publish": (st, [V, V, ctypes.c_char_p]),
        "kc_snapshot_bytes": (U64, [V]),
        "kc_snapshot_free": (None, [V]),
        "kc_capture_host": (st, [V, P(Dispatch), P(Region), SZ, ctypes.c_int, P(V), P(CaptureReport)]),
        "kc_host_arena_reserve": (st, [V, U64]),
        "kc_dev_arena_reserve": (st, [V, U64]),
        "kc_interpose_arm": (st, [V, ctypes.c_char_p, U64, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]),
        "kc_interpose_status": (st, [V, P(ctypes.c_int), P(U64), P(CaptureReport)]),
        "kc_interpose_take": (st, [V, P(V)]),
        "kc_interpose_arm_seq": (st, [V, ctypes.c_char_p, U64, U64, ctypes.c_int]),
        "kc_interpose_take_seq": (st, [V, P(V)]),
        "kc_snapshot_load": (st, [V, ctypes.c_char_p, ctypes.c_int, P(V)]),
        "kc_seq_load": (st, [V, ctypes.c_char_p, ctypes.c_int, P(V)]),
        "kc_snapshot_is_host": (ctypes.c_int, [V]),
        "kc_capture_incr": (st, [V, P(Dispatch), P(Region), SZ, ctypes.c_int, V, ctypes.c_int, P(V),
                                 P(CaptureReport)]),
        "kc_snapshot_shared_bytes": (U64, [V]),
        "kc_validate_module_vars": (st, [V, V, P(U64), P(U64)]),
        "kc_capture_seq": (st, [V, P(Dispatch), SZ, P(Region), SZ, ctypes.c_int, P(V), P(CaptureReport)]),
        "kc_seq_length": (SZ, [V]),
        "kc_seq_step": (V, [V, SZ]),
        "kc_seq_deps": (st, [V, P(ctypes.c_uint8), SZ]),
        "kc_seq_save": (st, [V, V, ctypes.c_char_p]),
        "kc_seq_free": (None, [V]),
        "kc_replay_seq": (st, [V, V, P(SeqReplayOpts), P(SeqStepReport), P(V)]),
        "kc_report_finalize": (st, [P(DiffReport), P(U64), P(I32), SZ]),
        "kc_peer_export": (st, [V, U64, P(I32), P(U64)]),
        "kc_peer_import": (st, [V, I32, I32, U64, U64, P(U64)]),
        "kc_peer_release": (st, [V, U64]),
        "kc_hash_plan_create": (st, [V, P(Region), SZ, P(V)]),
        "kc_hash_plan_run": (st, [V, V, V, V, V, V]),
        "kc_hash_plan_chunks": (U64, [V]),
        "kc_hash_plan_destroy": (st, [V]),
        "kc_diff_plan_create": (st, [V, P(Buffer), SZ, SZ, P(U64), P(U64), P(V)]),
        "kc_diff_plan_run": (st, [V, V, P(Tolerance), V, V, V]),
        "kc_diff_plan_destroy": (st, [V]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class HashPlan:
    """A prepared K1 region set (kc_hash_plan_*): run() is the launches alone."""

    def __init__(self, ctx: "Context", h: ctypes.c_void_p):
        self.ctx, self._h = ctx, h

    @property
    def chunks(self) -> int:
        return int(lib().kc_hash_plan_chunks(self._h))

    def run(self, d_chunk_hash: int, d_region_digest: int = 0, d_snapshot_digest: int = 0, stream: int = 0):
        self.ctx._check(lib().kc_hash_plan_run(self.ctx._h, self._h, d_chunk_hash or None, d_region_digest or None,
                                               d_snapshot_digest or None, stream or None), "kc_hash_plan_run")

    def close(self):
        if self._h:
            lib().kc_hash_plan_destroy(self._h)
            self._h = None


class DiffPlan:
    """A prepared K2 buffer set (kc_diff_plan_*): run() is the launches alone."""

    def __init__(self, ctx: "Context", h: ctypes.c_void_p):
        self.ctx, self._h = ctx, h

    def run(self, d_reports: int, d_bitmaps: int = 0, atol: float = 1e-8, rtol: float = 1e-5,
            equal_nan: bool = False, stream: int = 0):
        tol = Tolerance(atol, rtol, int(bool(equal_nan)), 0)
        self.ctx._check(lib().kc_diff_plan_run(self.ctx._h, self._h, ctypes.byref(tol), d_reports, d_bitmaps or None,
                                               stream or None), "kc_diff_plan_run")

    def close(self):
        if self._h:
            lib().kc_diff_plan_destroy(self._h)
            self._h = None


def status_name(s: int) -> str:
    try:
        return lib().kc_status_str(s).decode()
    except Exception:  # pragma: no cover - message path only
        return str(s)


def abi_version() -> int:
    return lib().kc_abi_version()


def build_info() -> str:
    return lib().kc_build_info().decode()


def count_chunks(regions: Sequence[Region]) -> int:
    arr = _regions(regions)
    return int(lib().kc_count_chunks(arr, len(regions)))


def report_finalize(rows, nbytes: Sequence[int], dtypes: Sequence[str]) -> list:
    """kc_report_finalize over reports merged across ranks (A9, C3).  ``rows``:
    an [R, 15] int64 array/tensor view of kc_diff_report structs (or raw
    bytes).  Returns the finalized reports as dicts (host only, no CUDA)."""
    import numpy as np
    raw = np.ascontiguousarray(np.asarray(rows, dtype=np.int64)).reshape(-1)
    n = len(nbytes)
    arr = (DiffReport * max(1, n))()
    ctypes.memmove(arr, raw.ctypes.data, min(raw.nbytes, ctypes.sizeof(DiffReport) * n))
    nb = (ctypes.c_uint64 * max(1, n))(*nbytes)
    dt = (ctypes.c_int32 * max(1, n))(*[DT[d] if isinstance(d, str) else int(d) for d in dtypes])
    rc = lib().kc_report_finalize(arr, nb, dt, n)
    if rc != KC_OK:
        raise KcError(rc, "kc_report_finalize: bad dtype or nbytes")
    return [arr[i].as_dict() for i in range(n)]


def region_array(regions) -> ctypes.Array:
    """Prebuilt kc_region array (reuse it across calls to keep marshalling off the hot path)."""
    return _regions(regions)


def buffer_array(bufs) -> ctypes.Array:
    """Prebuilt kc_buffer array (reuse it across calls)."""
    return Context._buffers(bufs)


def _regions(regions) -> ctypes.Array:
    if isinstance(regions, ctypes.Array) and regions._type_ is Region:
        return regions
    arr = (Region * max(1, len(regions)))()
    for i, r in enumerate(regions):
        if isinstance(r, Region):
            arr[i] = r
        else:  # (base, size) or (base, size, device, kind)
            t = tuple(r)
            arr[i] = Region(t[0], t[1], t[2] if len(t) > 2 else 0, t[3] if len(t) > 3 else 0, 0)
    return arr


def prereserve(snapshot_dir: str) -> tuple[int, bool]:
    """Pre-CUDA check that no host mapping overlaps the captured VA windows
    (the CUDA form of the paper's stage 2; R28).
    Returns (free windows, all free)."""
    n = ctypes.c_uint64(0)
    rc = lib().kc_prereserve(snapshot_dir.encode(), ctypes.byref(n))
    if rc < 0:
        raise KcError(rc, "kc_prereserve failed")
    return n.value, rc == KC_OK


def _reexec(argv: list, max_attempts: int) -> None:
    import os
    import sys
    attempt = int(os.environ.get("KC_REEXEC_ATTEMPT", "0"))
    if attempt + 1 < max_attempts:
        os.environ["KC_REEXEC_ATTEMPT"] = str(attempt + 1)
        os.execv(sys.executable, [sys.executable] + list(argv))


def exec_replay_process(argv: list, snapshot_dir: str, max_attempts: int = 16) -> None:
    """Call first thing in a replay process, before CUDA initialises: if a host
    mapping already sits on a captured VA window, re-exec for a new layout."""
    _, ok = prereserve(snapshot_dir)
    if not ok:
        _reexec(argv, max_attempts)


def restore_in_fresh_layout(ctx: "Context", snapshot_dir: str, argv: list, max_attempts: int = 16):
    """ctx.restore(); on KC_ERR_VA_UNAVAILABLE re-exec this process (ASLR gives
    the driver's VA arenas a new random placement) up to max_attempts times.
    The restore itself never relocates: it aborts and rolls back (R21)."""
    try:
        return ctx.restore(snapshot_dir)
    except KcError as e:
        if e.status == KC_ERR_VA_UNAVAILABLE:
            _reexec(argv, max_attempts)
            e.args = (f"{e.args[0] if e.args else ''} (after {max_attempts} process layouts)",)
        raise


def replay_seq_in_fresh_layout(ctx: "Context", seq: "Sequence", argv: list, max_attempts: int = 16, **kw):
    """ctx.replay_seq() with the same policy as restore_in_fresh_layout: a
    collision of the captured VAs with this process's driver arenas re-execs it."""
    try:
        return ctx.replay_seq(seq, **kw)
    except KcError as e:
        if e.status == KC_ERR_VA_UNAVAILABLE:
            _reexec(argv, max_attempts)
        raise


@dataclass
class Restored:
    handle: int
    ctx: "Context"

    def regions(self) -> list:
        n = ctypes.c_size_t(0)
        lib().kc_restored_regions(self.handle, None, 0, ctypes.byref(n))
        arr = (Region * max(1, n.value))()
        lib().kc_restored_regions(self.handle, arr, n.value, ctypes.byref(n))
        return [arr[i] for i in range(n.value)]

    def release(self):
        if self.handle:
            lib().kc_release(self.handle)
            self.handle = 0


@dataclass
class DevSnapshot:
    """An in-memory snapshot (F1): region bytes in an HBM arena (capture_dev) or
    a pinned host arena (capture_host)."""
    handle: int
    ctx: "Context"
    borrowed: bool = False   # a sequence step: owned by the kc_sequence

    def nbytes(self) -> int:
        return int(lib().kc_snapshot_bytes(self.handle))

    def is_host(self) -> bool:
        return bool(lib().kc_snapshot_is_host(self.handle))

    def shared_bytes(self) -> int:
        """Stored bytes referenced from base snapshots (incremental capture)."""
        return int(lib().kc_snapshot_shared_bytes(self.handle))

    def save(self, directory: str) -> None:
        self.ctx._check(lib().kc_snapshot_save(self.ctx.handle, self.handle, directory.encode()), "kc_snapshot_save")

    def publish(self, directory: str) -> None:
        """kc_snapshot_publish: metadata to `directory`, region bytes shared from this process's HBM (CUDA IPC)."""
        self.ctx._check(lib().kc_snapshot_publish(self.ctx.handle, self.handle, directory.encode()),
                        "kc_snapshot_publish")

    def free(self):
        if self.handle and not self.borrowed:
            lib().kc_snapshot_free(self.handle)
        self.handle = 0


class Sequence:
    """kc_sequence handle (F4 multi-kernel capture): one in-memory PRE_W snapshot per step."""

    def __init__(self, handle: int, ctx: "Context"):
        self.handle, self.ctx = handle, ctx

    def __len__(self) -> int:
        return int(lib().kc_seq_length(self.handle))

    def step(self, k: int) -> "DevSnapshot":
        """Step k's snapshot, BORROWED (owned by the sequence: do not free it)."""
        h = lib().kc_seq_step(self.handle, k)
        if not h:
            raise IndexError(k)
        return DevSnapshot(h, self.ctx, borrowed=True)

    def deps(self) -> list:
        """n x n matrix: deps[j][i] = KC_DEP_* flags of step j on step i < j."""
        n = len(self)
        buf = (ctypes.c_uint8 * max(1, n * n))()
        self.ctx._check(lib().kc_seq_deps(self.handle, buf, n * n), "kc_seq_deps")
        return [[int(buf[j * n + i]) for i in range(n)] for j in range(n)]

    def save(self, directory: str) -> None:
        self.ctx._check(lib().kc_seq_save(self.ctx.handle, self.handle, directory.encode()), "kc_seq_save")

    def free(self):
        if self.handle:
            lib().kc_seq_free(self.handle)
            self.handle = None


class Context:
    """A kc_ctx on one device (primary CUDA context)."""

    def __init__(self, device: int = 0, io_chunk_bytes: int = 0, pinned_depth: int = 0,
                 alloc_mode: int = KC_ALLOC_VMM):
        L = lib()
        self._h = ctypes.c_void_p()
        opt = Options(io_chunk_bytes, pinned_depth, device, alloc_mode, 0)
        rc = L.kc_create(ctypes.byref(self._h), ctypes.byref(opt))
        if rc != KC_OK:
            raise KcError(rc, f"kc_create(device={device}) failed")
        self.device = device

    # -- plumbing
    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().kc_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def kernel_launches(self) -> int:
        return int(lib().kc_kernel_launches(self._h))

    def last_error(self) -> str:
        return lib().kc_last_error(self._h).decode(errors="replace")

    def _check(self, rc: int, what: str, ok=(KC_OK,)) -> int:
        if rc not in ok:
            raise KcError(rc, f"{what}: {self.last_error()}")
        return rc

    # -- A1
    def track(self, ev: int, base: int, size: int = 0, device: int = 0, kind: int = KC_KIND_MEMALLOC) -> int:
        return self._check(lib().kc_track(self._h, ev, base, size, device, kind), "kc_track")

    def regions(self) -> list:
        n = ctypes.c_size_t(0)
        self._check(lib().kc_regions(self._h, None, 0, ctypes.byref(n)), "kc_regions")
        arr = (Region * max(1, n.value))()
        self._check(lib().kc_regions(self._h, arr, n.value, ctypes.byref(n)), "kc_regions")
        return [arr[i] for i in range(n.value)]

    def alloc(self, size: int) -> int:
        p = ctypes.c_uint64(0)
        self._check(lib().kc_alloc(self._h, size, ctypes.byref(p)), "kc_alloc")
        return p.value

    def peer_export(self, base: int) -> tuple[int, int]:
        """kc_peer_export: (fd, mapped size) of a kc_alloc'd region, for kc_peer_import elsewhere."""
        fd, sz = ctypes.c_int32(-1), ctypes.c_uint64(0)
        self._check(lib().kc_peer_export(self._h, base, ctypes.byref(fd), ctypes.byref(sz)), "kc_peer_export")
        return fd.value, sz.value

    def peer_import(self, pid: int, fd: int, size: int, want_va: int = 0) -> int:
        """kc_peer_import: map another process's exported allocation here; returns its VA."""
        va = ctypes.c_uint64(0)
        self._check(lib().kc_peer_import(self._h, pid, fd, size, want_va, ctypes.byref(va)), "kc_peer_import")
        return va.value

    def peer_release(self, va: int) -> None:
        self._check(lib().kc_peer_release(self._h, va), "kc_peer_release")

    def free(self, dptr: int):
        self._check(lib().kc_free(self._h, dptr), "kc_free")

    def track_install(self):
        return self._check(lib().kc_track_install(self._h), "kc_track_install")

    def track_uninstall(self):
        return self._check(lib().kc_track_uninstall(self._h), "kc_track_uninstall")

    # -- K1 / K3 / K2
    def hash(self, regions, d_chunk_hash: int, d_region_digest: int = 0, d_snapshot_digest: int = 0,
             stream: int = 0, n: int | None = None):
        arr = _regions(regions)
        n = len(regions) if n is None else n
        self._check(lib().kc_hash(self._h, arr, n, d_chunk_hash or None, d_region_digest or None,
                                  d_snapshot_digest or None, stream or None), "kc_hash")

    def hash_plan(self, regions) -> "HashPlan":
        """kc_hash_plan_create: the region set validated and uploaded once (run it many times)."""
        arr = _regions(regions)
        h = ctypes.c_void_p()
        self._check(lib().kc_hash_plan_create(self._h, arr, len(regions), ctypes.byref(h)), "kc_hash_plan_create")
        return HashPlan(self, h)

    def diff_plan(self, bufs, n_reports: int, report_nbytes: Sequence[int],
                  bitmap_word0: Sequence[int] | None = None) -> "DiffPlan":
        """kc_diff_plan_create: the buffer set (as kc_diff_async) validated and uploaded once."""
        arr = self._buffers(bufs)
        rn = (ctypes.c_uint64 * max(1, n_reports))(*report_nbytes)
        w0 = (ctypes.c_uint64 * max(1, n_reports))(*bitmap_word0) if bitmap_word0 is not None else None
        h = ctypes.c_void_p()
        self._check(lib().kc_diff_plan_create(self._h, arr, len(bufs), n_reports, rn, w0, ctypes.byref(h)),
                    "kc_diff_plan_create")
        return DiffPlan(self, h)

    def written(self, d_pre: int, d_post: int, n_chunks: int, d_bitmap: int, d_count: int = 0, stream: int = 0):
        self._check(lib().kc_written(self._h, d_pre, d_post, n_chunks, d_bitmap, d_count or None, stream or None),
                    "kc_written")

    @staticmethod
    def _buffers(bufs) -> ctypes.Array:
        if isinstance(bufs, ctypes.Array) and bufs._type_ is Buffer:
            return bufs
        arr = (Buffer * max(1, len(bufs)))()
        for i, b in enumerate(bufs):
            if isinstance(b, Buffer):
                arr[i] = b
            else:  # (ref, act, nbytes, dtype[, report[, chunk0]])
                t = tuple(b)
                dt = DT[t[3]] if isinstance(t[3], str) else int(t[3])
                arr[i] = Buffer(t[0], t[1], t[2], dt, t[4] if len(t) > 4 else i, t[5] if len(t) > 5 else 0)
        return arr

    def diff(self, bufs, atol: float = 1e-8, rtol: float = 1e-5, equal_nan: bool = False, stream: int = 0,
             with_bitmaps: bool = True):
        """K2 over (ref, act, nbytes, dtype) device buffers -> (list of report dicts, list of bitmap word lists)."""
        n = len(bufs)
        arr = self._buffers(bufs)
        reps = (DiffReport * max(1, n))()
        words = [((b.nbytes + KC_CHUNK_BYTES - 1) // KC_CHUNK_BYTES + 63) // 64 for b in arr[:n]]
        bm = (ctypes.c_uint64 * max(1, sum(words)))()
        tol = Tolerance(atol, rtol, int(bool(equal_nan)), 0)
        self._check(lib().kc_diff(self._h, arr, n, ctypes.byref(tol), reps, bm if with_bitmaps else None,
                                  stream or None), "kc_diff")
        out_b, o = [], 0
        for w in words:
            out_b.append([bm[o + k] for k in range(w)])
            o += w
        return [reps[i].as_dict() for i in range(n)], out_b

    def validate_host_ref(self, bufs, ref_manifest_ptr: int, atol: float = 1e-8, rtol: float = 1e-5,
                          equal_nan: bool = False, stream: int = 0, with_bitmaps: bool = True,
                          d_act_manifest: int = 0):
        """kc_validate_host_ref over (host ref address, device act VA, nbytes, dtype) buffers and a host
        reference manifest (address of the u64 chunk hashes; 0 = byte-exact mode, every reference byte
        crosses PCIe) -> (reports, bitmaps, h2d bytes)."""
        n = len(bufs)
        arr = self._buffers(bufs)
        reps = (DiffReport * max(1, n))()
        words = [((b.nbytes + KC_CHUNK_BYTES - 1) // KC_CHUNK_BYTES + 63) // 64 for b in arr[:n]]
        bm = (ctypes.c_uint64 * max(1, sum(words)))()
        tol = Tolerance(atol, rtol, int(bool(equal_nan)), 0)
        moved = ctypes.c_uint64(0)
        self._check(lib().kc_validate_host_ref(self._h, arr, n, ref_manifest_ptr or None, ctypes.byref(tol), reps,
                                               bm if with_bitmaps else None, d_act_manifest or None,
                                               ctypes.byref(moved), stream or None), "kc_validate_host_ref")
        out_b, o = [], 0
        for w in words:
            out_b.append([bm[o + k] for k in range(w)])
            o += w
        return [reps[i].as_dict() for i in range(n)], out_b, int(moved.value)

    def diff_async(self, bufs, n_reports: int, report_nbytes: Sequence[int], d_reports: int,
                   bitmap_word0: Sequence[int] | None = None, d_bitmaps: int = 0, atol: float = 1e-8,
                   rtol: float = 1e-5, equal_nan: bool = False, stream: int = 0):
        arr = self._buffers(bufs)
        rn = report_nbytes if isinstance(report_nbytes, ctypes.Array) else \
            (ctypes.c_uint64 * max(1, n_reports))(*report_nbytes)
        w0 = None
        if bitmap_word0 is not None:
            w0 = bitmap_word0 if isinstance(bitmap_word0, ctypes.Array) else \
                (ctypes.c_uint64 * max(1, n_reports))(*bitmap_word0)
        tol = Tolerance(atol, rtol, int(bool(equal_nan)), 0)
        self._check(lib().kc_diff_async(self._h, arr, len(bufs), n_reports, rn, w0, ctypes.byref(tol), d_reports,
                                        d_bitmaps or None, stream or None), "kc_diff_async")

    def hash_diff_async(self, bufs, d_chunk_hash: int, d_reports: int, d_bitmaps: int = 0, d_dirty: int = 0,
                        atol: float = 1e-8, rtol: float = 1e-5, equal_nan: bool = False, stream: int = 0):
        """kc_hash_diff_async (F2): K5 hashes every act buffer while comparing it with its
        ref; K2 then diffs only the dirty chunks.  One report per buffer."""
        arr = self._buffers(bufs)
        tol = Tolerance(atol, rtol, int(bool(equal_nan)), 0)
        self._check(lib().kc_hash_diff_async(self._h, arr, len(bufs), ctypes.byref(tol), d_chunk_hash, d_reports,
                                             d_bitmaps or None, d_dirty or None, stream or None), "kc_hash_diff_async")

    # -- closure
    def capture(self, directory: str, *, image: bytes | None = None, mangled: str | None = None, grid=(1, 1, 1),
                block=(1, 1, 1), smem: int = 0, kernarg: bytes = b"", regions=None, mode: int = KC_MODE_PRE_W,
                stream: int = 0, func: int = 0, cluster=None) -> tuple[int, dict]:
        """kc_capture.  func: a CUfunction handle of the application's own module
        (then image may be omitted when kc_track_install recorded the module's load)."""
        d, keep = self._dispatch(image, mangled, grid, block, smem, kernarg, stream, func, cluster)
        rep = CaptureReport()
        arr = _regions(regions) if regions is not None else None
        rc = lib().kc_capture(self._h, ctypes.byref(d), arr, len(regions) if regions is not None else 0,
                              directory.encode(), mode, ctypes.byref(rep))
        self._check(rc, "kc_capture", ok=(KC_OK, KC_PARTIAL))
        return rc, rep.as_dict()

    def _dispatch(self, image, mangled, grid, block, smem, kernarg, stream, func=0, cluster=None,
                  cooperative=False):
        img = ctypes.create_string_buffer(image, len(image)) if image else None
        ka = ctypes.create_string_buffer(kernarg, len(kernarg)) if kernarg else None
        d = Dispatch(func or None, ctypes.cast(img, ctypes.c_void_p) if img else None, len(image) if image else 0,
                     mangled.encode() if mangled else None, (ctypes.c_uint32 * 3)(*grid),
                     (ctypes.c_uint32 * 3)(*block), smem, len(kernarg), ctypes.cast(ka, ctypes.c_void_p) if ka else None,
                     stream or None, (ctypes.c_uint32 * 3)(*(tuple(cluster) + (1,) * (3 - len(cluster))))
                     if cluster else (ctypes.c_uint32 * 3)(0, 0, 0), 1 if cooperative else 0)
        return d, (img, ka)

    def capture_dev(self, *, image: bytes | None = None, mangled: str | None = None, grid=(1, 1, 1),
                    block=(1, 1, 1), smem: int = 0, kernarg: bytes = b"", regions=None, mode: int = KC_MODE_PRE_W,
                    stream: int = 0, host: bool = False, base: "DevSnapshot | None" = None, func: int = 0,
                    cluster=None, cooperative: bool = False) -> tuple[DevSnapshot, dict]:
        """kc_capture into a device arena (F1), or a pinned host arena (host=True:
        kc_capture_host); with base=, only chunks changed against it are copied
        (kc_capture_incr); cluster = thread-block cluster dims of a cluster launch."""
        d, keep = self._dispatch(image, mangled, grid, block, smem, kernarg, stream, func, cluster, cooperative)
        rep = CaptureReport()
        h = ctypes.c_void_p()
        arr = _regions(regions) if regions is not None else None
        nreg = len(regions) if regions is not None else 0
        if base is not None:
            name = "kc_capture_incr"
            rc = lib().kc_capture_incr(self._h, ctypes.byref(d), arr, nreg, mode, base.handle, int(host),
                                       ctypes.byref(h), ctypes.byref(rep))
        else:
            name = "kc_capture_host" if host else "kc_capture_dev"
            rc = getattr(lib(), name)(self._h, ctypes.byref(d), arr, nreg, mode, ctypes.byref(h), ctypes.byref(rep))
        self._check(rc, name, ok=(KC_OK, KC_PARTIAL))
        return DevSnapshot(h.value, self), rep.as_dict()

    def capture_host(self, **kw) -> tuple[DevSnapshot, dict]:
        """kc_capture_host: the capture into a pinned host arena."""
        return self.capture_dev(host=True, **kw)

    def interpose_arm(self, target: str | None, index: int = 0, directory: str | None = None,
                      mode: int = KC_MODE_PRE_W, host: bool = False) -> None:
        """kc_interpose_arm: capture launch `index` of a kernel whose name contains `target` (CUPTI hook)."""
        self._check(lib().kc_interpose_arm(self._h, target.encode() if target else None, index,
                                           directory.encode() if directory else None, mode, int(host)),
                    "kc_interpose_arm")

    def interpose_status(self) -> dict:
        st, seen, rep = ctypes.c_int(0), ctypes.c_uint64(0), CaptureReport()
        rc = lib().kc_interpose_status(self._h, ctypes.byref(st), ctypes.byref(seen), ctypes.byref(rep))
        return {"rc": rc, "state": st.value, "seen": seen.value, "report": rep.as_dict(),
                "error": self.last_error() if rc < 0 else ""}

    def load_snapshot(self, directory: str, host: bool = False) -> "DevSnapshot":
        """kc_snapshot_load: a kc-snapshot/1 directory into device (or pinned host) memory."""
        h = ctypes.c_void_p()
        self._check(lib().kc_snapshot_load(self._h, directory.encode(), int(host), ctypes.byref(h)),
                    "kc_snapshot_load")
        return DevSnapshot(h.value, self)

    def load_seq(self, directory: str, host: bool = False) -> "Sequence":
        """kc_seq_load: a kc-sequence/1 directory back into memory."""
        h = ctypes.c_void_p()
        self._check(lib().kc_seq_load(self._h, directory.encode(), int(host), ctypes.byref(h)), "kc_seq_load")
        return Sequence(h.value, self)

    def interpose_arm_seq(self, target: str | None, first: int, count: int, host: bool = False) -> None:
        """kc_interpose_arm_seq: capture launches [first, first+count) of `target` as a sequence (F4)."""
        self._check(lib().kc_interpose_arm_seq(self._h, target.encode() if target else None, first, count, int(host)),
                    "kc_interpose_arm_seq")

    def interpose_take_seq(self) -> "Sequence":
        h = ctypes.c_void_p()
        self._check(lib().kc_interpose_take_seq(self._h, ctypes.byref(h)), "kc_interpose_take_seq")
        return Sequence(h.value, self)

    def interpose_take(self) -> "DevSnapshot":
        h = ctypes.c_void_p()
        self._check(lib().kc_interpose_take(self._h, ctypes.byref(h)), "kc_interpose_take")
        return DevSnapshot(h.value, self)

    def dev_arena_reserve(self, nbytes: int) -> None:
        """kc_dev_arena_reserve: map a device arena ahead of time and park it (0 releases it)."""
        self._check(lib().kc_dev_arena_reserve(self._h, nbytes), "kc_dev_arena_reserve")

    def host_arena_reserve(self, nbytes: int) -> None:
        """kc_host_arena_reserve: pin a host arena ahead of time (0 frees the parked one)."""
        self._check(lib().kc_host_arena_reserve(self._h, nbytes), "kc_host_arena_reserve")

    def restore_dev(self, snap: DevSnapshot) -> tuple[Restored, dict]:
        h = ctypes.c_void_p()
        rep = RestoreReport()
        rc = lib().kc_restore_dev(self._h, snap.handle, ctypes.byref(h), ctypes.byref(rep))
        if rc != KC_OK:
            e = KcError(rc, f"kc_restore_dev: {self.last_error()}")
            e.report = rep.as_dict()
            raise e
        return Restored(h.value, self), rep.as_dict()

    def restore_dev_into(self, snap: DevSnapshot, restored: Restored) -> dict:
        """kc_restore_dev_into: the snapshot restored over a live restore of the same regions."""
        rep = RestoreReport()
        rc = lib().kc_restore_dev_into(self._h, snap.handle, restored.handle, ctypes.byref(rep))
        if rc != KC_OK:
            e = KcError(rc, f"kc_restore_dev_into: {self.last_error()}")
            e.report = rep.as_dict()
            raise e
        return rep.as_dict()

    def restore(self, directory: str) -> tuple[Restored, dict]:
        h = ctypes.c_void_p()
        rep = RestoreReport()
        rc = lib().kc_restore(self._h, directory.encode(), ctypes.byref(h), ctypes.byref(rep))
        if rc != KC_OK:
            e = KcError(rc, f"kc_restore: {self.last_error()}")
            e.report = rep.as_dict()
            raise e
        return Restored(h.value, self), rep.as_dict()

    def replay(self, restored: Restored, iterations: int = 1, no_recopy: bool = False, dump_dir: str | None = None,
               image_override: bytes | None = None, stream: int = 0, grid=None, block=None, smem: int | None = None,
               symbol: str | None = None) -> dict:
        """kc_replay; grid/block/smem/symbol override the captured launch shape (a retuned variant)."""
        ov = ctypes.create_string_buffer(image_override, len(image_override)) if image_override else None
        o = ReplayOpts(iterations, int(no_recopy), dump_dir.encode() if dump_dir else None,
                       ctypes.cast(ov, ctypes.c_void_p) if ov else None, len(image_override) if image_override else 0,
                       stream or None)
        if grid is not None:
            o.overrides |= 1
            o.grid[:] = list(grid) + [1] * (3 - len(grid))
        if block is not None:
            o.overrides |= 2
            o.block[:] = list(block) + [1] * (3 - len(block))
        if smem is not None:
            o.overrides |= 4
            o.smem_bytes = smem
        if symbol is not None:
            o.overrides |= 8
            o.symbol = symbol.encode()
        rep = ReplayReport()
        self._check(lib().kc_replay(self._h, restored.handle, ctypes.byref(o), ctypes.byref(rep)), "kc_replay")
        return rep.as_dict()

    def capture_seq(self, dispatches: Sequence[dict], regions=None, host: bool = False
                    ) -> tuple["Sequence", list]:
        """kc_capture_seq: dispatches = [dict(image=, mangled=, grid=, block=, smem=, kernarg=, stream=, func=)]."""
        keep = []
        arr = (Dispatch * len(dispatches))()
        for i, d in enumerate(dispatches):
            arr[i], k = self._dispatch(d.get("image"), d.get("mangled"), d.get("grid", (1, 1, 1)),
                                       d.get("block", (1, 1, 1)), d.get("smem", 0), d.get("kernarg", b""),
                                       d.get("stream", 0), d.get("func", 0), d.get("cluster"))
            keep.append(k)
        reps = (CaptureReport * len(dispatches))()
        h = ctypes.c_void_p()
        rg = _regions(regions) if regions is not None else None
        rc = lib().kc_capture_seq(self._h, arr, len(dispatches), rg, len(regions) if regions is not None else 0,
                                  int(host), ctypes.byref(h), reps)
        self._check(rc, "kc_capture_seq", ok=(KC_OK, KC_PARTIAL))
        return Sequence(h.value, self), [r.as_dict() for r in reps]

    def replay_seq(self, seq: "Sequence", first: int = 0, count: int | None = None, overrides=None,
                   atol: float = 1e-8, rtol: float = 1e-5, equal_nan: bool = False, stream: int = 0,
                   keep: bool = False):
        """kc_replay_seq: joint replay of steps [first, first+count); overrides = list of code objects
        (bytes or None) per replayed step.  Returns (step reports, Restored or None)."""
        n = len(seq)
        count = n - first if count is None else count
        bufs = [ctypes.create_string_buffer(b, len(b)) if b else None for b in (overrides or [])]
        ov = None
        if overrides is not None:
            ov = (ctypes.c_void_p * max(1, count))(*[ctypes.cast(b, ctypes.c_void_p) if b else None for b in bufs])
        o = SeqReplayOpts(first, count, ov, None, Tolerance(atol, rtol, int(bool(equal_nan)), 0), stream or None)
        reps = (SeqStepReport * max(1, count))()
        h = ctypes.c_void_p()
        self._check(lib().kc_replay_seq(self._h, seq.handle, ctypes.byref(o), reps, ctypes.byref(h) if keep else None),
                    "kc_replay_seq")
        return [reps[i].as_dict() for i in range(count)], (Restored(h.value, self) if keep else None)

    def validate_module_vars(self, restored: Restored) -> tuple[int, int]:
        """F3: (variables checked, variables differing from their captured post value) of the last replay."""
        n, m = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(lib().kc_validate_module_vars(self._h, restored.handle, ctypes.byref(n), ctypes.byref(m)),
                    "kc_validate_module_vars")
        return int(n.value), int(m.value)

    def validate(self, restored: Restored, outs=None, atol: float = 1e-8, rtol: float = 1e-5,
                 equal_nan: bool = False) -> tuple[list, int]:
        tol = Tolerance(atol, rtol, int(bool(equal_nan)), 0)
        cap = 4096
        reps = (DiffReport * cap)()
        nrep = ctypes.c_size_t(0)
        unexpected = ctypes.c_uint64(0)
        arr = None
        n = 0
        if outs is not None:
            arr = (Buffer * max(1, len(outs)))()
            for i, (act, nbytes, dt) in enumerate(outs):
                arr[i] = Buffer(0, act, nbytes, DT[dt] if isinstance(dt, str) else int(dt), i, 0)
            n = len(outs)
        self._check(lib().kc_validate(self._h, restored.handle, arr, n, ctypes.byref(tol), reps, cap,
                                      ctypes.byref(nrep), ctypes.byref(unexpected)), "kc_validate")
        return [reps[i].as_dict() for i in range(min(cap, nrep.value))], unexpected.value


def exported_symbols() -> list:
    """Names of the C ABI entry points (checked against include/kc.h in the CPU tests)."""
    return list(EXPORTED)
