"""Subprocess worker: CUPTI driver-API interposition (A1).
Prints one JSON line describing what the tracker saw."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_03208_b200 import kc  # noqa: E402


def main():
    out = {}
    ctx = kc.Context(0)
    ctx.track_install()
    try:
        ctx.track_install()
        out["double_install"] = "accepted"
    except kc.KcError as e:
        out["double_install"] = e.status
    from cuda.bindings import driver as drv
    # 1. a raw driver allocation
    err, p = drv.cuMemAlloc(3 << 20)
    p = int(p)
    regs = {r.base: r for r in ctx.regions()}
    out["memalloc_tracked"] = p in regs and regs[p].size == 3 << 20 and regs[p].kind == kc.KC_KIND_MEMALLOC
    # 2. VMM through kc_alloc: cuMemMap is intercepted (kc_alloc does not double-feed)
    v = ctx.alloc(5 << 20)
    regs = {r.base: r for r in ctx.regions()}
    out["vmm_tracked"] = v in regs and regs[v].kind == kc.KC_KIND_VMM
    out["vmm_size"] = regs[v].size if v in regs else None
    # 3. torch's caching allocator (cudaMalloc -> driver allocation)
    import torch
    t = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    tp = t.data_ptr()
    regs = ctx.regions()
    out["torch_segment_tracked"] = any(r.base <= tp < r.base + r.size for r in regs)
    # 4. frees are seen
    drv.cuMemFree(p)
    ctx.free(v)
    regs = {r.base: r for r in ctx.regions()}
    out["memalloc_free_seen"] = p not in regs
    out["vmm_unmap_seen"] = v not in regs
    # 5. async pool allocation
    err, s = drv.cuStreamCreate(0)
    err, q = drv.cuMemAllocAsync(1 << 20, s)
    drv.cuStreamSynchronize(s)
    regs = {r.base: r for r in ctx.regions()}
    out["pool_tracked"] = int(q) in regs and regs[int(q)].kind == kc.KC_KIND_POOL
    drv.cuMemFreeAsync(q, s)
    drv.cuStreamSynchronize(s)
    out["pool_free_seen"] = int(q) not in {r.base for r in ctx.regions()}
    ctx.track_uninstall()
    err, p2 = drv.cuMemAlloc(1 << 20)
    out["untracked_after_uninstall"] = int(p2) not in {r.base for r in ctx.regions()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
