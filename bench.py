#!/usr/bin/env python
"""bench.py -- snapshot hash+validate throughput of the Kerncap address-space
closure hot path on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1; NCCL)

Workload (default): config c4, the 30,074,000,000-byte vLLM-style MoE pool of
185 regions (24 x w13 + 24 x w2 bf16 expert stacks, 24 pointer tables, 113
misc regions), E1 residency-first placement over the N GPUs.
One STEP is one pass of the whole device hot path over the pool:
  A2  K1 pre-manifest (XXH64 per 64 KiB chunk + region/snapshot digests)
  A3  the target dispatch (F3, pointer-indirected MoE GEMV through ptr_table)
  A4  K1 post-manifest + K3 written set
  A8  K2 validate: restored/replayed pool vs captured reference pool, per region
  A9  (N > 1) NCCL all_gather of manifests + all_reduce of the reports
value = algorithmic HBM bytes of the hash and diff kernels per second, whole
job (2 x pool for the two hashes + 2 x pool for the diff), inputs resident in
HBM and larger than L2.  e2e = the same metric with the step's snapshot bytes
copied host->device (pinned) every step and the reports read back.
e2e_host_ref = the host-resident reference validated by kc_validate_host_ref
(only the manifest and the reference chunks whose hash differs cross PCIe).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "snapshot hash+validate GB/s (1/2/4/8 B200, % HBM peak); 30 GB capture->replay latency"
UNIT = "GB/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons polled through NVML every 5 ms DURING the
    timed region (the data of B200_PROFILING.md's nvidia-smi clocks line)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples, self.reasons = [], 0
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # reported in the JSON
            self.err = repr(e)[:120]

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: " + getattr(self, "err", "")]}
        self.stop_ev.set()
        self.t.join()
        sm = sorted(self.samples)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": sm[0] if sm else None,
                "reasons": sorted(n for b, n in self.REASONS.items() if self.reasons & b),
                "samples": len(sm), "source": "nvml, 5 ms poll during the timed steps"}


# ------------------------------------------------------------------ workload
class Pool:
    """This rank's shard of the c4 pool: live regions, the captured reference copy, the F3 dispatch."""

    def __init__(self, ctx, rank, world, device, log, plant=False, placement="e1"):
        import numpy as np
        import torch
        import synth
        self.torch = torch
        self.ctx = ctx
        self.placement = placement
        specs = synth.c4_specs()
        owner = synth.c4_placement(specs, world) if placement == "e1" else [0] * len(specs)
        # the F3 activations/output sit with layer 0 on rank 0 (its closure is local)
        for i, s in enumerate(specs):
            if s.name in ("x", "topk", "y"):
                owner[i] = 0
        self.specs = [s for s, o in zip(specs, owner) if o == rank]
        self.total_bytes = sum(s.size for s in specs)
        gen = torch.Generator(device=f"cuda:{device}")
        self.va, self.ref = {}, {}
        t0 = time.time()
        for s in self.specs:
            self.va[s.name] = ctx.alloc(s.size)
        for idx, s in enumerate(specs):
            if s.name not in self.va:
                continue
            v = synth.dev_view(self.va[s.name], s.size, device)
            gen.manual_seed(synth.seed(4, 100 + idx))
            if s.fill == "ptr_table":
                layer = s.layer
                t = synth.c4_ptr_table(self.va[f"w13_{layer}"], self.va[f"w2_{layer}"])
                v.copy_(torch.from_numpy(t.view(np.uint8)))
            elif s.fill == "topk":
                v.zero_()
                tk = synth.c4_topk()
                v[: tk.nbytes].copy_(torch.from_numpy(tk.view(np.uint8).reshape(-1)))
            else:
                synth.fill_device(v, s, gen)
        torch.cuda.synchronize()
        log(f"rank {rank}: {len(self.specs)} regions, {sum(s.size for s in self.specs) / 1e9:.3f} GB filled in "
            f"{time.time() - t0:.1f}s")
        # hashing order: ascending VA at N = 1 (so the snapshot digest is defined);
        # global spec order at N > 1 (VAs of different processes are not comparable)
        self.gidx = {s.name: i for i, s in enumerate(specs)}
        self.all_specs, self.owner = specs, owner
        if world == 1:
            self.specs.sort(key=lambda s: self.va[s.name])
        else:
            self.specs.sort(key=lambda s: self.gidx[s.name])
        self.regions = [(self.va[s.name], s.size) for s in self.specs]
        self.bytes = sum(s.size for s in self.specs)
        self.dtype_of = {self.va[s.name]: s.dtype for s in self.specs}
        # F3 dispatch (rank 0): the target kernel, loaded like any captured code object
        self.fn = None
        if "x" in self.va:
            from cuda.bindings import driver as drv
            image = open(synth.FIXTURE_CUBIN, "rb").read()
            err, self.mod = drv.cuModuleLoadData(image)
            err, self.fn = drv.cuModuleGetFunction(self.mod, b"kc_fixture_moe_gemv")
            self.image = image
            self.kernarg = synth.c4_kernarg(self.va["ptr_0"], self.va["x"], self.va["topk"], self.va["y"])
        self.launch_f3(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        # the captured reference (post-dispatch) copy of every region: "what the replay must reproduce"
        for s in self.specs:
            self.ref[s.name] = ctx.alloc(s.size)
            synth.dev_view(self.ref[s.name], s.size, device).copy_(synth.dev_view(self.va[s.name], s.size, device))
        torch.cuda.synchronize()
        self.n_plants = 0
        if plant:
            self.n_plants = self.plant(device)
        self.C = None
        if placement == "e2":
            self.share_e2(ctx, rank, world, log)

    def share_e2(self, ctx, rank, world, log):
        """E2: the whole pool lives in rank 0's HBM; every rank maps
        rank 0's live and reference regions (kc_peer_export -> kc_peer_import: NVLink
        peer access from the other GPUs) and hashes/diffs a contiguous, 64-chunk
        aligned share of the global chunk range (global spec order), so bitmap words
        of different ranks are disjoint."""
        import torch.distributed as dist
        objs = [None]
        if rank == 0:
            objs[0] = {"pid": os.getpid(),
                       "va": {n: (va,) + ctx.peer_export(va) for n, va in self.va.items()},
                       "ref": {n: (va,) + ctx.peer_export(va) for n, va in self.ref.items()}}
        dist.broadcast_object_list(objs, src=0)
        ex = objs[0]
        t0 = time.time()
        if rank != 0:
            self.va = {n: ctx.peer_import(ex["pid"], fd, sz, va) for n, (va, fd, sz) in ex["va"].items()}
            self.ref = {n: ctx.peer_import(ex["pid"], fd, sz, va) for n, (va, fd, sz) in ex["ref"].items()}
        dist.barrier()
        specs = self.all_specs
        nck = [(sp.size + 65535) // 65536 for sp in specs]
        C = sum(nck)
        bnd = [min(C, (C * r // world) // 64 * 64) for r in range(world)] + [C]
        lo, hi = bnd[rank], bnd[rank + 1]
        self.e2_counts = [bnd[r + 1] - bnd[r] for r in range(world)]
        self.sub = []   # (global idx, chunk offset in the region, nbytes) of this rank's share
        off = 0
        for g, sp in enumerate(specs):
            a, b = max(lo, off), min(hi, off + nck[g])
            if a < b:
                k0 = a - off
                self.sub.append((g, k0, min(sp.size, b * 65536 - off * 65536) - k0 * 65536))
            off += nck[g]
        self.regions = [(self.va[specs[g].name] + 65536 * k0, n) for g, k0, n in self.sub]
        self.bytes = sum(n for _, _, n in self.sub)
        log(f"rank {rank}: E2 share chunks [{lo}, {hi}) of {C} over {len(self.sub)} sub-regions, "
            f"{self.bytes / 1e9:.3f} GB of rank 0's pool ({'own HBM' if rank == 0 else 'peer-mapped'}; "
            f"mapped in {time.time() - t0:.2f}s)")

    def plant(self, device) -> int:
        """--plant: XOR single bytes of the reference copy at offsets fixed by the
        region's global index (the same at every N): a 1-ULP step, a sign flip and
        an exponent-bit flip in one of every 7 bf16 regions.  Each plant changes
        exactly one byte."""
        import synth
        n = 0
        for s in self.specs:
            g = self.gidx[s.name]
            if s.dtype != "bf16" or g % 7 != 3:
                continue
            v = synth.dev_view(self.ref[s.name], s.size, device)
            ne = s.size // 2
            offs = {}
            for k, (lohi, mask) in enumerate(((0, 0x01), (1, 0x80), (1, 0x01))):
                e = (g * 2654435761 + k * 40503 * 32768 + 17) % ne
                offs[2 * e + lohi] = mask
            for off, mask in offs.items():
                v[off] ^= mask
                n += 1
        self.torch.cuda.synchronize()
        return n

    def launch_f3(self, stream):
        if self.fn is None:
            return 0
        import ctypes
        from cuda.bindings import driver as drv
        import synth
        warps = synth.C4_T * 2816
        args = ((self.va["ptr_0"], self.va["x"], self.va["topk"], self.va["y"], synth.C4_T, 2816, 2048),
                (ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                 ctypes.c_int))
        err, = drv.cuLaunchKernel(self.fn, (warps * 32 + 255) // 256, 1, 1, 256, 1, 1, 0, stream, args, 0)
        assert int(err) == 0, err
        return 1

    def diff_buffers(self):
        """(buffers, report sizes, report bitmap word offsets).  E1: one report per
        local region.  E2: one report per GLOBAL region (185), each rank's share a
        segment of it starting at its chunk offset (bitmap_chunk0)."""
        from paper_2605_03208_b200 import kc
        out = []
        if self.placement == "e2":
            specs = self.all_specs
            for g, k0, n in self.sub:
                s = specs[g]
                out.append(kc.Buffer(self.ref[s.name] + 65536 * k0, self.va[s.name] + 65536 * k0, n, kc.DT[s.dtype],
                                     g, k0))
            sizes = [s.size for s in specs]
        else:
            for i, s in enumerate(self.specs):
                out.append(kc.Buffer(self.ref[s.name], self.va[s.name], s.size, kc.DT[s.dtype], i, 0))
            sizes = [s.size for s in self.specs]
        word0, acc = [], 0
        for n in sizes:
            word0.append(acc)
            acc += ((n + 65535) // 65536 + 63) // 64
        return out, sizes, word0, acc


def workload_config(world: int) -> dict:
    """The `config` both arms print (the reference arm times a bounded sample of it)."""
    import synth
    return {"workload": "c4: vLLM-style MoE weight pool, 30,074,000,000 B, 185 regions, E1 placement",
            "step": "K1 pre-manifest + F3 dispatch + K1 post-manifest + K3 written set + K2 pool-pair validate"
                    + (" + NCCL combine" if world > 1 else ""),
            "alg_bytes_per_step": 4 * synth.C4_TOTAL, "pool_bytes": synth.C4_TOTAL, "regions": 185,
            "l2": "inputs (30 GB) >> L2 (126 MB); no flush needed",
            "parallelism": f"E1 residency-first shards over {world} GPU(s)"}


def run_ours(a, rank, world, device, log):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_03208_b200 import kc

    torch.cuda.set_device(device)
    ctx = kc.Context(device)
    pool = Pool(ctx, rank, world, device, log, plant=a.plant, placement=a.placement)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    C = kc.count_chunks(pool.regions)
    nreg = len(pool.regions)
    pre = torch.zeros(max(1, C), dtype=torch.int64, device="cuda")
    post = torch.zeros_like(pre)
    dig = torch.zeros(max(1, nreg) + 1, dtype=torch.int64, device="cuda")
    words = (C + 63) // 64
    wbm = torch.zeros(max(1, words), dtype=torch.int64, device="cuda")
    wcnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    bufs, rep_nbytes, word0, acc = pool.diff_buffers()
    n_rep = len(rep_nbytes)
    REP_WORDS = 15  # sizeof(kc_diff_report) / 8
    reps = torch.zeros(max(1, n_rep) * REP_WORDS, dtype=torch.int64, device="cuda")
    bms = torch.zeros(max(1, acc), dtype=torch.int64, device="cuda")
    KEYS = ("hash_pre", "dispatch", "hash_post", "written", "diff", "combine")
    evs = [{k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in KEYS}
           for _ in range(a.steps)]

    # A9 combine (N > 1): C1 plan broadcast once; per step C2 manifests all-gather, C3 reports all-reduce
    plan = perm = None
    glob_reps = None
    e2 = pool.placement == "e2"
    if world > 1:
        from paper_2605_03208_b200 import dist as kd
        specs_all = pool.all_specs
        plan = kd.Plan.from_rank0(list(range(len(specs_all))) if rank == 0 else None,
                                  [s.size for s in specs_all] if rank == 0 else None,
                                  pool.owner if rank == 0 else None, device="cuda")
        perm = plan.manifest_permutation().cuda()
        bperm = plan.bitmap_permutation().cuda()
        rows = torch.tensor([pool.gidx[s.name] for s in pool.specs], dtype=torch.int64, device="cuda")
        glob_reps = torch.zeros(len(specs_all), REP_WORDS, dtype=torch.int64, device="cuda")
        glob = {}
        peer = None
        if a.combine == "peer" and not e2:
            # the combine fused into the producing kernels over peer memory: rank 0 owns the
            # global manifest, report rows and bitmap words ([world, pad] layouts); every rank
            # maps them (kc_peer_export -> kc_peer_import) and its K1 stores the post-manifest,
            # and its K2 accumulates reports and sets bitmap bits, straight into its slice of
            # rank 0's HBM (NVLink on a multi-GPU node).  The exchange is then a barrier.
            import synth
            pad = max(1, plan.max_local_chunks())
            maxrows = max(1, max(sum(1 for o in plan.owner if o == r) for r in range(world)))
            padw = max(1, max(plan.bitmap_words(r) for r in range(world)))
            sizes = {"man": world * pad * 8, "reps": world * maxrows * 8 * REP_WORDS, "bms": world * padw * 8}
            objs = [None]
            if rank == 0:
                bases = {k: ctx.alloc(n) for k, n in sizes.items()}
                objs[0] = {"pid": os.getpid(), "buf": {k: (va,) + ctx.peer_export(va) for k, va in bases.items()}}
            dist.broadcast_object_list(objs, src=0)
            if rank == 0:
                peer_va = bases
            else:
                peer_va = {k: ctx.peer_import(objs[0]["pid"], fd, sz, va) for k, (va, fd, sz) in objs[0]["buf"].items()}
            dist.barrier()
            peer = {"va": peer_va, "pad": pad, "maxrows": maxrows, "padw": padw}
            # this rank's slices, as tensors aliasing rank 0's memory (the step code is unchanged)
            post = synth.dev_view(peer_va["man"] + 8 * rank * pad, 8 * max(1, C), device).view(torch.int64)
            reps = synth.dev_view(peer_va["reps"] + 8 * REP_WORDS * rank * maxrows,
                                  8 * REP_WORDS * max(1, n_rep), device).view(torch.int64)
            bms = synth.dev_view(peer_va["bms"] + 8 * rank * padw, 8 * max(1, acc), device).view(torch.int64)
            log(f"rank {rank}: peer combine: manifest, reports and bitmaps written into rank 0's HBM "
                f"({'own' if rank == 0 else 'peer-mapped'})")

    def step(ev):
        launches = 0

        def rec(k, i):
            if ev is not None:
                ev[k][i].record(stream)
        rec("hash_pre", 0)
        ctx.hash(pool.regions, pre.data_ptr(), dig.data_ptr(), dig.data_ptr() + 8 * nreg if world == 1 else 0,
                 stream=sh)
        rec("hash_pre", 1)
        rec("dispatch", 0)
        launches += pool.launch_f3(sh)
        rec("dispatch", 1)
        rec("hash_post", 0)
        ctx.hash(pool.regions, post.data_ptr(), stream=sh)
        rec("hash_post", 1)
        rec("written", 0)
        ctx.written(pre.data_ptr(), post.data_ptr(), C, wbm.data_ptr(), wcnt.data_ptr(), stream=sh)
        rec("written", 1)
        rec("diff", 0)
        ctx.diff_async(bufs, n_rep, rep_nbytes, reps.data_ptr(), word0, bms.data_ptr(), stream=sh)
        rec("diff", 1)
        if world > 1:
            rec("combine", 0)
            if peer is not None:   # the results are already in rank 0's HBM: make them visible
                stream.synchronize()
                dist.barrier()
            elif e2:   # contiguous chunk ranges; every rank reports all 185 regions (its segments)
                glob["manifest"] = kd.gather_ranges(post, pool.e2_counts)              # C2
                glob["reports"] = kd.combine_reports(reps.view(-1, REP_WORDS))          # C3
                glob["bitmaps"] = kd.gather_bitmaps(bms)                                # C4 (disjoint words)
            else:
                glob["manifest"] = kd.Plan.gather_manifest(plan, post, perm)            # C2
                glob_reps.zero_()
                glob_reps.index_copy_(0, rows, reps.view(-1, REP_WORDS))
                glob["reports"] = kd.combine_reports(glob_reps)                         # C3
                glob["bitmaps"] = kd.gather_region_bitmaps(plan, bms, bperm)            # C4
            rec("combine", 1)
        return launches

    for _ in range(a.warmup):
        step(None)
    torch.cuda.synchronize()
    # correctness gate before timing: the replayed pool must validate bit-exactly
    rh = reps.view(-1, REP_WORDS).cpu().numpy()
    chk = torch.tensor([int(rh[:, 3].sum()), pool.n_plants], dtype=torch.int64, device="cuda")
    if world > 1:   # (E2: a region's plants may lie in another rank's share)
        kd._all_reduce(chk, dist.ReduceOp.SUM)
    assert int(chk[0]) == int(chk[1]), \
        f"pool pair: {int(chk[0])} differing bytes, {int(chk[1])} planted: validation failed"

    l0 = ctx.kernel_launches()
    clocks = ClockSampler(device)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    f3 = 0
    for i in range(a.steps):
        f3 += step(evs[i])
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = ctx.kernel_launches() - l0 + f3
    ms_local = e0.elapsed_time(e1) / a.steps
    tsum = {k: 0.0 for k in KEYS}
    for ev in evs:
        for k in KEYS:
            if k == "combine" and world == 1:
                continue
            tsum[k] += ev[k][0].elapsed_time(ev[k][1])
    tmax = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    alg_local = 4 * pool.bytes
    alg = torch.tensor([float(alg_local)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(alg)
    ms = float(tmax.item())
    value = float(alg.item()) / (ms * 1e-3) / 1e9

    # cross-N fingerprint (O7: N-GPU results equal the 1-GPU ones bit for bit): SHA-256 of the
    # post-manifest in global spec order (pointer tables excluded: they hold this process's
    # VAs), of the finalized reports (kc_report_finalize) and of the per-region bitmaps, all in
    # global spec order -- at N > 1 the C2/C3/C4 results of the last timed step
    import hashlib
    import numpy as np
    specs_all = pool.all_specs
    nck = [(s.size + 65535) // 65536 for s in specs_all]
    nwd = [(c + 63) // 64 for c in nck]
    if world > 1 and peer is not None:   # rank 0 reads the combined results from its own HBM
        gman = synth.dev_view(peer["va"]["man"], 8 * world * peer["pad"], device).view(torch.int64)
        glob["manifest"] = gman[perm]
        grep = synth.dev_view(peer["va"]["reps"], 8 * REP_WORDS * world * peer["maxrows"],
                              device).view(torch.int64).view(world * peer["maxrows"], REP_WORDS)
        ridx = []
        seen = [0] * world
        for o in plan.owner:   # global spec order -> (owner, its local row)
            ridx.append(o * peer["maxrows"] + seen[o])
            seen[o] += 1
        glob["reports"] = grep[torch.tensor(ridx, dtype=torch.int64, device="cuda")]
        gbm = synth.dev_view(peer["va"]["bms"], 8 * world * peer["padw"], device).view(torch.int64)
        pw = max(1, max(plan.bitmap_words(r) for r in range(world)))
        assert pw == peer["padw"]
        glob["bitmaps"] = gbm[bperm]
    if world > 1:
        gm = glob["manifest"].cpu().numpy()
        rep_rows = glob["reports"].cpu().numpy()
        gb = glob["bitmaps"].cpu().numpy()
        starts = np.cumsum([0] + nck[:-1])
        wst = np.cumsum([0] + nwd[:-1])
        pieces = [gm[starts[g]:starts[g] + nck[g]] for g in range(len(specs_all))]
        bm_pieces = [gb[wst[g]:wst[g] + nwd[g]] for g in range(len(specs_all))]
    else:
        hp, bh = post.cpu().numpy(), bms.cpu().numpy()
        rl = reps.view(-1, REP_WORDS).cpu().numpy()
        byg, bmg, o = {}, {}, 0
        rep_rows = np.zeros((len(specs_all), REP_WORDS), dtype=np.int64)
        for i, s in enumerate(pool.specs):
            g = pool.gidx[s.name]
            byg[g] = hp[o:o + nck[g]]
            o += nck[g]
            bmg[g] = bh[word0[i]:word0[i] + nwd[g]]
            rep_rows[g] = rl[i]
        pieces = [byg[g] for g in range(len(specs_all))]
        bm_pieces = [bmg[g] for g in range(len(specs_all))]
    fin = kc.report_finalize(rep_rows, [s.size for s in specs_all], [s.dtype for s in specs_all])
    counters = [sum(r[k] for r in fin) for k in ("differing_bytes", "differing_elems", "nan_ref", "nan_act",
                                                 "allclose_fail")]
    fp = hashlib.sha256()
    for s, pc in zip(specs_all, pieces):
        if not s.name.startswith("ptr_"):
            fp.update(pc.tobytes())
    fingerprint = {"post_manifest_sha256_excl_ptr_tables": fp.hexdigest(),
                   "reports_sha256": hashlib.sha256(json.dumps(fin, sort_keys=True).encode()).hexdigest(),
                   "bitmaps_sha256": hashlib.sha256(b"".join(b.tobytes() for b in bm_pieces)).hexdigest(),
                   "bitmap_bits": int(sum(bin(int(w) & 0xFFFFFFFFFFFFFFFF).count("1") for b in bm_pieces for w in b)),
                   "max_ulp": max(r["max_ulp"] for r in fin), "max_abs": max(r["max_abs"] for r in fin),
                   "max_rel": max(r["max_rel"] for r in fin),
                   "chunks": int(sum(p.size for p in pieces)), "report_counter_sums": [int(x) for x in counters]}

    # per-kernel roofline: the dominant kernel by time share
    per = {k: tsum[k] / a.steps for k in tsum}
    k1_ms = (per["hash_pre"] + per["hash_post"]) / 2
    k2_ms = per["diff"]
    peak, peak_src = peaks()
    kern = {
        "K1_hash": {"ms": k1_ms, "alg_bytes": pool.bytes, "gbs": pool.bytes / (k1_ms * 1e-3) / 1e9},
        "K2_diff": {"ms": k2_ms, "alg_bytes": 2 * pool.bytes, "gbs": 2 * pool.bytes / (k2_ms * 1e-3) / 1e9},
        "K3_written_ms": per["written"], "F3_dispatch_ms": per["dispatch"],
    }
    if world > 1:
        kern["A9_combine_ms"] = per["combine"]
    dom = "K2_diff" if k2_ms >= 2 * k1_ms else "K1_hash"   # K1 runs twice per step (pre and post)
    dom_ms = k2_ms if dom == "K2_diff" else 2 * k1_ms
    share = dom_ms / ms if ms else None
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):  # dram__bytes_read.sum + dram__bytes_write.sum per launch, one ncu --set full capture
        t = json.load(open(tp)).get(dom)
        if t and t.get("alg_bytes_per_launch") == kern[dom]["alg_bytes"]:
            traffic, traffic_src = t["dram_bytes_per_launch"], t["source"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak, "unit": "GB/s",
            "frac": kern[dom]["gbs"] / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peak_src,
            "frac_of_spec_8000": kern[dom]["gbs"] / 8000.0, "share_of_step": share,
            "alg_bytes_per_launch": kern[dom]["alg_bytes"]}

    # ------------------------------------------------------------------ F2 fused step
    fused = None
    if not a.no_fused and not e2:
        fused = run_fused(a, ctx, pool, stream, pre, post, dig, wbm, wcnt, bufs, reps, C, nreg, world, log)

    # ------------------------------------------------------------------ e2e
    e2e = e2e_host_ref = None
    if not a.no_e2e and not e2:
        e2e_host_ref = run_e2e_host_ref(a, ctx, pool, stream, world, log, pre, post, dig, wbm, wcnt, C, nreg)
        torch.cuda.synchronize()
        torch._C._host_emptyCache()   # pinned e2e staging back to the OS
        e2e = run_e2e(a, ctx, pool, stream, world, log, pre, post, dig, wbm, wcnt, C, nreg)
        torch.cuda.synchronize()
        torch._C._host_emptyCache()
    lat = None
    if world == 1 and not a.no_latency:
        try:
            lat = run_latency(a, ctx, pool, log)
        except Exception as ex:  # reported, never hidden
            lat = {"error": repr(ex)[:300]}

    # PCIe roofline (A5 D2H capture, A6 H2D restore, the e2e H2D): rates over the in-run
    # measured pinned peak (best of 5 x 1 GiB) and the 64 GB/s Gen5 x16 spec
    pcie = None
    if lat and "host_pinned" in lat and "pcie" in lat["host_pinned"]:
        pk = lat["host_pinned"]["pcie"]

        def prow(gbs, peak_key):
            return {"achieved": gbs, "peak_measured": pk[peak_key], "frac": gbs / pk[peak_key],
                    "frac_of_spec_64": gbs / 64.0}
        pcie = {"unit": "GB/s", "measured": pk,
                "d2h_capture_host_pinned": prow(lat["host_pinned"]["copy_out_gbs"], "d2h_gbs"),
                "h2d_restore_host_pinned": prow(lat["host_pinned"]["copy_in_gbs"], "h2d_gbs")}
        if e2e:
            pcie["h2d_e2e_byte_exact"] = prow(e2e["h2d_gbs"], "h2d_gbs")
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded; bf16 N(0,0.02) expert weights, bf16 misc, device-pointer tables)",
        "config": workload_config(world),
        "shard": {"regions_this_rank": len(pool.regions), "bytes_this_rank": pool.bytes,
                  "alg_bytes_per_step_all_ranks": int(float(alg.item()))},
        "roofline": roof, "kernels": kern, "clocks": clk, "gpu_launches": launches,
        "e2e": e2e, "e2e_host_ref": e2e_host_ref, "capture_replay": lat, "pcie": pcie, "fingerprint": fingerprint,
        "fused_step": fused,
    }
    return res, pool


def run_fused(a, ctx, pool, stream, pre, post, dig, wbm, wcnt, bufs, reps, C, nreg, world, log):
    """F2: the same step with the post-manifest and the pool-pair validation fused
    (kc_hash_diff_async: K5 reads pool and reference once, hashing the pool while
    comparing; K2 then reads only dirty chunks).  Same algorithmic work as the
    headline step (hash 2N, validate 2N); the post-manifest and the reports must
    equal the unfused step's bit for bit."""
    import torch
    sh = stream.cuda_stream
    post_ref = post.clone()
    reps_ref = reps.clone()
    reps_f = torch.zeros_like(reps)
    dirty = torch.zeros((C + 63) // 64 + 1, dtype=torch.int64, device="cuda")
    bms = torch.zeros(sum(((b.nbytes + 65535) // 65536 + 63) // 64 for b in bufs) + 1, dtype=torch.int64,
                      device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]

    def step(ev):
        ctx.hash(pool.regions, pre.data_ptr(), dig.data_ptr(), dig.data_ptr() + 8 * nreg if world == 1 else 0,
                 stream=sh)
        n = pool.launch_f3(sh)
        if ev is not None:
            ev[0].record(stream)
        ctx.hash_diff_async(bufs, post.data_ptr(), reps_f.data_ptr(), bms.data_ptr(), dirty.data_ptr(), stream=sh)
        if ev is not None:
            ev[1].record(stream)
        ctx.written(pre.data_ptr(), post.data_ptr(), C, wbm.data_ptr(), wcnt.data_ptr(), stream=sh)
        return n
    for _ in range(a.warmup):
        step(None)
    torch.cuda.synchronize()
    same = bool(torch.equal(post, post_ref)) and bool(torch.equal(reps_f, reps_ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(a.steps):
        step(evs[i])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
    ms = float(tm.item())
    k5_ms = sum(x[0].elapsed_time(x[1]) for x in evs) / a.steps
    n_dirty = int(sum(bin(int(w) & 0xFFFFFFFFFFFFFFFF).count("1") for w in dirty.cpu().tolist()))
    log(f"fused step: {ms:.3f} ms (K5 + filtered K2 {k5_ms:.3f} ms, {n_dirty} dirty chunks), "
        f"bit-identical to the unfused step: {same}")
    return {"ms_per_step": ms, "value_same_metric": 4 * pool.bytes * world / (ms * 1e-3) / 1e9,
            "identical_to_unfused": same, "dirty_chunks": n_dirty,
            "K5_plus_filtered_K2": {"ms": k5_ms, "hbm_bytes": 2 * pool.bytes,
                                    "gbs": 2 * pool.bytes / (k5_ms * 1e-3) / 1e9},
            "step": "K1 pre-manifest + F3 dispatch + K5 fused post-manifest/compare + K2 over dirty chunks + "
                    "K3 written set"}


def run_e2e_host_ref(a, ctx, pool, stream, world, log, pre, post, dig, wbm, wcnt, C, nreg):
    """The metric end to end through the public API with the captured reference in
    pinned HOST memory (a host-resident snapshot: its bytes and its manifest).
    Every step: K1 pre-manifest, the F3 dispatch, kc_validate_host_ref (one K5
    pass over the live pool gives the post-manifest and the Inf/NaN chunks; the
    reference manifest goes host->device, chunks whose hash differs have their
    reference bytes copied host->device, K2 runs over exactly those; reports and
    bitmaps come back to the host), K3 written set.  The result is bit-identical
    to the device step's (checked below); h2d/d2h bytes are what actually moved."""
    import torch
    import synth
    host = {}
    for s in pool.specs:
        h = torch.empty(s.size, dtype=torch.uint8, pin_memory=True)
        h.copy_(synth.dev_view(pool.ref[s.name], s.size, torch.cuda.current_device()))
        host[s.name] = h
    # the snapshot's manifest (computed when the reference was captured), pinned host
    man_dev = torch.zeros(max(1, C), dtype=torch.int64, device="cuda")
    ctx.hash([(pool.ref[s.name], s.size) for s in pool.specs], man_dev.data_ptr())
    torch.cuda.synchronize()
    man_host = man_dev.cpu().pin_memory()
    del man_dev
    hbufs = [(host[s.name].data_ptr(), pool.va[s.name], s.size, s.dtype) for s in pool.specs]
    sh = stream.cuda_stream
    out = {}

    def step():
        ctx.hash(pool.regions, pre.data_ptr(), dig.data_ptr(), dig.data_ptr() + 8 * nreg if world == 1 else 0,
                 stream=sh)
        pool.launch_f3(sh)
        reps, bms, moved = ctx.validate_host_ref(hbufs, man_host.data_ptr(), d_act_manifest=post.data_ptr(),
                                                 stream=sh)
        ctx.written(pre.data_ptr(), post.data_ptr(), C, wbm.data_ptr(), wcnt.data_ptr(), stream=sh)
        out["reps"], out["moved"], out["bm_words"] = reps, moved, sum(len(b) for b in bms)
    for _ in range(max(1, a.warmup)):
        step()
    torch.cuda.synchronize()
    ok = all(r["differing_bytes"] == 0 and r["pass"] == 1 for r in out["reps"])
    steps = a.steps
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
    ms = float(tm.item())
    host.clear()
    nw = (C + 63) // 64
    d2h = 120 * len(hbufs) + 8 * out["bm_words"] + 16 * nw
    total = 4 * pool.total_bytes
    log(f"e2e (host-resident reference, kc_validate_host_ref): {ms:.3f} ms/step, h2d {out['moved'] / 1e6:.2f} MB/step, "
        f"validated {ok}")
    return {"value": total / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": out["moved"],
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": steps, "validated_bit_exact": ok,
            "path": "kc_hash (pre) + F3 dispatch + kc_validate_host_ref (K5 post-manifest over the live pool, "
                    "H2D of the reference manifest and of reference chunks whose hash differs, K2 over those and "
                    "over Inf/NaN chunks) + kc_written; reports and bitmaps read back every step",
            "note": "unchanged chunks are recognised by XXH64 equality with the snapshot's manifest (DESIGN.md "
                    "R34, the same test as the written set W) instead of a byte compare, so this is not the "
                    "headline e2e; `e2e` copies every reference byte and compares all of them"}


def run_e2e(a, ctx, pool, stream, world, log, pre, post, dig, wbm, wcnt, C, nreg):
    """The metric end to end through the public C ABI with the captured snapshot in
    pinned HOST memory (what kc_capture_host leaves behind): every step runs the K1
    pre-manifest, the F3 dispatch, kc_validate_host_ref in BYTE-EXACT mode (every
    reference byte crosses PCIe through the library's 3 x 256 MiB staging ring on its
    copy stream, K2 diffs each piece as it lands, K1 gives the post-manifest; the
    reports and bitmaps come back to the host) and K3.  Same algorithmic work as
    the device step (2 hashes of N, a diff reading 2N) plus N bytes host->device."""
    import torch
    import synth
    host = {}
    for s in pool.specs:
        h = torch.empty(s.size, dtype=torch.uint8, pin_memory=True)
        h.copy_(synth.dev_view(pool.ref[s.name], s.size, torch.cuda.current_device()))
        host[s.name] = h
    torch.cuda.synchronize()
    hbufs = [(host[s.name].data_ptr(), pool.va[s.name], s.size, s.dtype) for s in pool.specs]
    sh = stream.cuda_stream
    out = {}

    def step():
        ctx.hash(pool.regions, pre.data_ptr(), dig.data_ptr(), dig.data_ptr() + 8 * nreg if world == 1 else 0,
                 stream=sh)
        pool.launch_f3(sh)
        reps, bms, moved = ctx.validate_host_ref(hbufs, 0, d_act_manifest=post.data_ptr(), stream=sh)
        ctx.written(pre.data_ptr(), post.data_ptr(), C, wbm.data_ptr(), wcnt.data_ptr(), stream=sh)
        out["reps"], out["moved"], out["bm_words"] = reps, moved, sum(len(b) for b in bms)
    step()   # warm-up: plan caches, the staging ring, its events
    torch.cuda.synchronize()
    diffs = sum(r["differing_bytes"] for r in out["reps"])
    ok = diffs == pool.n_plants if pool.n_plants else all(r["differing_bytes"] == 0 and r["pass"] == 1
                                                          for r in out["reps"])
    steps = max(1, a.e2e_steps)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    ms = e0.elapsed_time(e1) / steps
    tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(tm, op=torch.distributed.ReduceOp.MAX)
    ms = float(tm.item())
    host.clear()
    total = 4 * pool.total_bytes
    d2h = 120 * len(hbufs) + 8 * out["bm_words"]
    log(f"e2e (byte-exact kc_validate_host_ref): {ms:.2f} ms/step, h2d {out['moved'] / 1e9:.2f} GB/step "
        f"({out['moved'] / (ms * 1e-3) / 1e9:.1f} GB/s), validated {ok}")
    return {"value": total / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": out["moved"],
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "wall_ms_per_step": 1e3 * wall, "steps": steps,
            "h2d_gbs": out["moved"] / (ms * 1e-3) / 1e9, "validated_bit_exact": bool(ok),
            "path": "kc_hash (pre) + F3 dispatch + kc_validate_host_ref(ref_manifest=NULL: byte-exact, every "
                    "reference byte H2D through the library's staging ring overlapped with K2; K1 post-manifest) "
                    "+ kc_written; reports and bitmaps read back every step"}


def run_latency(a, ctx, pool, log):
    """The metric's second half: 30 GB capture -> replay latency through the public
    C ABI, per stage, for both snapshot sinks.
      device (F1): kc_capture_dev (K1 pre-manifest, D2D copy of every region into an
        HBM arena, the F3 dispatch, K1 post-manifest, W) -> the live regions are
        freed -> kc_restore_dev maps them back at the captured VAs, copies the arena
        in and verifies the manifest -> kc_replay -> kc_validate.
      host_pinned: kc_capture_host (the same, D2H into a pinned host arena at PCIe
        rate) -> kc_restore_dev (H2D) -> kc_replay -> kc_validate.
      host_pinned_incremental: kc_capture_incr against that snapshot (only chunks
        whose hash changed cross PCIe) -> kc_restore_dev -> kc_replay -> kc_validate.
      files: kc_capture (PRE_W, pinned D2H by 8 I/O threads into /dev/shm) ->
        kc_restore from the files -> kc_replay -> kc_validate.
    Each run's restored memory serves as the live state of the next."""
    import shutil
    import torch
    import synth
    from paper_2605_03208_b200 import kc
    regions = [(b, n) for b, n in pool.regions]
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    warps = synth.C4_T * 2816
    disp = dict(image=image, mangled="kc_fixture_moe_gemv", grid=((warps * 32 + 255) // 256, 1, 1),
                block=(256, 1, 1), kernarg=pool.kernarg, regions=regions, mode=kc.KC_MODE_PRE_W)
    ys = [s for s in pool.specs if s.name == "y"][0]
    out = {}

    def finish(name, cap, rst, r, times):
        rep = ctx.replay(r)
        t4 = time.perf_counter()
        reps, unexpected = ctx.validate(r)
        t5 = time.perf_counter()
        ok = (all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0
              and rst["verify_mismatch_chunks"] == 0 and cap["written_chunks"] > 0 and len(reps) > 0)
        same = sorted((x.base, x.size) for x in r.regions()) == sorted(regions)
        t0, t1, t2, t3 = times
        total = (t1 - t0) + (t3 - t2) + (t4 - t3) + (t5 - t4)
        log(f"capture->replay [{name}]: capture {t1 - t0:.3f}s restore {t3 - t2:.3f}s replay {t4 - t3:.4f}s "
            f"validate {t5 - t4:.4f}s ok={ok}")
        return {"latency_s": total, "validated_bit_exact": bool(ok), "same_vas": bool(same),
                "written_chunks": cap["written_chunks"],
                "stages_s": {"capture_total": t1 - t0, "capture_hash_pre": cap["t_hash_pre_s"],
                             "capture_copy": cap["t_d2h_s"], "capture_dispatch": cap["t_dispatch_s"],
                             "capture_hash_post": cap["t_hash_post_s"], "restore_total": t3 - t2,
                             "restore_reserve_map": rst["t_reserve_s"], "restore_copy_in": rst["t_h2d_s"],
                             "restore_verify": rst["t_verify_s"], "replay": t4 - t3, "validate": t5 - t4},
                "copy_out_gbs": (cap["d2h_bytes"] or pool.bytes) / max(cap["t_d2h_s"], 1e-9) / 1e9,
                "copy_out_bytes": cap["d2h_bytes"] or pool.bytes,
                "copy_in_gbs": rst["h2d_bytes"] / max(rst["t_h2d_s"], 1e-9) / 1e9}

    # ---- device sink (F1): a cold cycle (first in-memory capture and VMM restore
    # of this process: lazy kernel loading, first arena and physical allocations)
    # and a warm one on the restored state; both reported, the warm one is the
    # steady-state latency of a resident tool
    torch.cuda.empty_cache()          # earlier stages' cached blocks back to the driver
    cold = None
    r_dev = None
    for cycle in ("cold", "warm"):
        synth.dev_view(pool.va["y"], ys.size).zero_()   # a fresh output buffer: the dispatch writes W != {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        snap, cap = ctx.capture_dev(**disp)
        t1 = time.perf_counter()
        if r_dev is None:
            for s in pool.specs:
                ctx.free(pool.va[s.name])
        else:
            r_dev.release()
        t2 = time.perf_counter()
        r_dev, rst = ctx.restore_dev(snap)
        t3 = time.perf_counter()
        res = finish(f"device {cycle}", cap, rst, r_dev, (t0, t1, t2, t3))
        res["arena_bytes"] = snap.nbytes()
        snap.free()
        if cycle == "cold":
            cold = res
    out["device"] = res
    out["device"]["cycle"] = "warm (second capture -> restore in this process)"
    out["device"]["cold"] = {"latency_s": cold["latency_s"], "stages_s": cold["stages_s"],
                             "validated_bit_exact": cold["validated_bit_exact"]}

    # ---- device sink, restore in place (kc_restore_dev_into): the resident tool's repeated
    # capture -> replay cycle keeps the restore's VA windows and mappings and only copies the
    # snapshot back over them (stage 5 without stages 2-4); two cycles, the second reported
    try:
        for cycle in ("first", "second"):
            synth.dev_view(pool.va["y"], ys.size).zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            snap, cap = ctx.capture_dev(**disp)
            t1 = time.perf_counter()
            t2 = time.perf_counter()
            rst = ctx.restore_dev_into(snap, r_dev)
            t3 = time.perf_counter()
            res = finish(f"device in place ({cycle})", cap, rst, r_dev, (t0, t1, t2, t3))
            snap.free()
        res["cycle"] = "second kc_capture_dev -> kc_restore_dev_into over the live restore"
        out["device_inplace"] = res
    except Exception as ex:  # reported, never hidden
        out["device_inplace"] = {"error": repr(ex)[:300], "validated_bit_exact": False}

    # ---- device arena published to a fresh replay process (CUDA IPC): the
    # paper's workflow (capture in the application, replay in another process)
    # without the bytes leaving HBM
    try:
        out["device_ipc"] = run_ipc_sink(a, ctx, pool, disp, ys, log)
    except Exception as ex:  # reported, never hidden
        out["device_ipc"] = {"error": repr(ex)[:300], "validated_bit_exact": False}

    # ---- pinned host sink (the restored memory is now the live state); the arena
    # is pinned ahead of time like the staging ring, its cost reported apart
    tp = time.perf_counter()
    ctx.host_arena_reserve(pool.bytes + 256 * len(regions))
    pin_s = time.perf_counter() - tp
    synth.dev_view(pool.va["y"], ys.size).zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    snap, cap = ctx.capture_host(**disp)
    t1 = time.perf_counter()
    r_dev.release()
    t2 = time.perf_counter()
    r_host, rst = ctx.restore_dev(snap)
    t3 = time.perf_counter()
    out["host_pinned"] = finish("host_pinned", cap, rst, r_host, (t0, t1, t2, t3))
    out["host_pinned"]["arena_bytes"] = snap.nbytes()
    out["host_pinned"]["arena_pin_s"] = pin_s
    out["host_pinned"]["pcie"] = pcie_peak(log)

    # ---- F2 incremental capture against that snapshot: only chunks whose hash changed are copied
    synth.dev_view(pool.va["y"], ys.size).zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    snap_i, cap = ctx.capture_host(base=snap, **disp)
    t1 = time.perf_counter()
    r_host.release()
    t2 = time.perf_counter()
    r_host, rst = ctx.restore_dev(snap_i)
    t3 = time.perf_counter()
    out["host_pinned_incremental"] = finish("host_pinned_incremental", cap, rst, r_host, (t0, t1, t2, t3))
    out["host_pinned_incremental"]["copied_bytes"] = snap_i.nbytes()
    out["host_pinned_incremental"]["shared_bytes"] = snap_i.shared_bytes()
    snap_i.free()
    snap.free()
    ctx.host_arena_reserve(0)

    # ---- file sink
    d = a.latency_dir
    shutil.rmtree(d, ignore_errors=True)
    synth.dev_view(pool.va["y"], ys.size).zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc, cap = ctx.capture(d, **disp)
    t1 = time.perf_counter()
    r_host.release()
    t2 = time.perf_counter()
    r, rst = ctx.restore(d)
    t3 = time.perf_counter()
    out["files"] = finish("files", cap, rst, r, (t0, t1, t2, t3))
    out["files"]["sink"] = d
    r.release()
    # capture once, replay many: the file snapshot loaded into HBM once
    # (kc_snapshot_load, verified), then each edit -> replay -> validate
    # iteration restores from memory instead of re-reading 30 GB of files
    try:
        tl0 = time.perf_counter()
        snap_l = ctx.load_snapshot(d)
        tl1 = time.perf_counter()
        r2, rst2 = ctx.restore_dev(snap_l)
        tl2 = time.perf_counter()
        cap_l = dict(cap, t_hash_pre_s=0.0, t_d2h_s=0.0, t_dispatch_s=0.0, t_hash_post_s=0.0, d2h_bytes=0)
        it = finish("files loaded to HBM", cap_l, rst2, r2, (tl1, tl1, tl1, tl2))
        out["files_loaded"] = {"load_s": tl1 - tl0, "load_gbs": pool.bytes / (tl1 - tl0) / 1e9,
                               "iteration_s": it["latency_s"], "validated_bit_exact": it["validated_bit_exact"],
                               "same_vas": it["same_vas"], "stages_s": it["stages_s"],
                               "note": "one kc_snapshot_load of the file snapshot, then restore -> replay -> "
                                       "validate per iteration (the paper's edit-replay loop)"}
        r2.release()
        snap_l.free()
    except Exception as ex:  # reported, never hidden
        out["files_loaded"] = {"error": repr(ex)[:300], "validated_bit_exact": False}
    shutil.rmtree(d, ignore_errors=True)
    out["bytes"] = pool.bytes
    out["latency_s"] = out["device"]["latency_s"]
    out["validated_bit_exact"] = all(out[k]["validated_bit_exact"]
                                     for k in ("device", "device_ipc", "host_pinned", "host_pinned_incremental",
                                               "files", "files_loaded"))
    return out


def run_ipc_sink(a, ctx, pool, disp, ys, log):
    """kc_capture_dev + kc_snapshot_publish here; kc_restore (CUDA IPC copy-in at
    the captured VAs) + kc_replay + kc_validate in a fresh process, timed inside
    it.  latency = capture + the child's restore + replay + validate; the
    child's interpreter start, CUDA init and exit are reported apart."""
    import shutil
    import subprocess
    import torch
    import synth
    d = a.latency_dir + "_ipc"
    shutil.rmtree(d, ignore_errors=True)
    synth.dev_view(pool.va["y"], ys.size).zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    snap, cap = ctx.capture_dev(**disp)
    t1 = time.perf_counter()
    snap.publish(d)
    t2 = time.perf_counter()
    p = subprocess.run([sys.executable, os.path.abspath(__file__), "--replay-child", d], capture_output=True,
                       text=True, timeout=600, env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get(
                           "CUDA_VISIBLE_DEVICES", str(torch.cuda.current_device()))))
    t3 = time.perf_counter()
    snap.free()
    shutil.rmtree(d, ignore_errors=True)
    for x in p.stderr.splitlines():
        if x.startswith("[kc]"):
            log("  child " + x)
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    if p.returncode != 0 or not lines:
        raise RuntimeError(f"replay child failed rc={p.returncode}: {p.stderr[-400:]}")
    ch = json.loads(lines[-1])
    lat = (t1 - t0) + ch["restore_s"] + ch["replay_s"] + ch["validate_s"]
    log(f"capture->replay [device_ipc]: capture {t1 - t0:.3f}s (publish {t2 - t1:.3f}s) | fresh process: restore "
        f"{ch['restore_s']:.3f}s replay {ch['replay_s']:.4f}s validate {ch['validate_s']:.4f}s ok={ch['ok']} "
        f"(child wall {t3 - t2:.1f}s incl. interpreter + CUDA init)")
    return {"latency_s": lat, "validated_bit_exact": bool(ch["ok"]), "same_vas": bool(ch["same_vas"]),
            "written_chunks": cap["written_chunks"],
            "stages_s": {"capture_total": t1 - t0, "capture_hash_pre": cap["t_hash_pre_s"],
                         "capture_copy": cap["t_d2h_s"], "capture_hash_post": cap["t_hash_post_s"],
                         "publish": t2 - t1, "restore_total": ch["restore_s"], **ch["restore_stages"],
                         "replay": ch["replay_s"], "validate": ch["validate_s"]},
            "copy_in_gbs": ch["copy_in_gbs"], "child_wall_s": t3 - t2, "child_attempts": ch["attempts"],
            "note": "restore/replay/validate timed inside the fresh replay process; its startup excluded"}


def replay_child(d):
    """--replay-child DIR: a fresh process restoring a published snapshot."""
    from paper_2605_03208_b200 import kc
    kc.exec_replay_process(sys.argv, d)          # pre-CUDA VA collision check (re-exec on collision)
    ctx = kc.Context(0)
    t0 = time.perf_counter()
    r, rst = kc.restore_in_fresh_layout(ctx, d, sys.argv)
    t1 = time.perf_counter()
    ctx.replay(r)
    t2 = time.perf_counter()
    reps, unexpected = ctx.validate(r)
    t3 = time.perf_counter()
    import json as _j
    regs = json.load(open(os.path.join(d, "memory_regions.json")))
    same = sorted((x.base, x.size) for x in r.regions()) == sorted((int(e["base"], 16), int(e["size"])) for e in regs)
    ok = all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0 and rst["verify_mismatch_chunks"] == 0 \
        and len(reps) > 0
    print(_j.dumps({"restore_s": t1 - t0, "replay_s": t2 - t1, "validate_s": t3 - t2, "ok": ok, "same_vas": same,
                    "restore_stages": {"restore_reserve_map": rst["t_reserve_s"], "restore_copy_in": rst["t_h2d_s"],
                                       "restore_verify": rst["t_verify_s"]},
                    "copy_in_gbs": rst["h2d_bytes"] / max(rst["t_h2d_s"], 1e-9) / 1e9,
                    "attempts": int(os.environ.get("KC_REEXEC_ATTEMPT", "0")) + 1}))
    r.release()
    ctx.close()


def pcie_peak(log, nbytes: int = 1 << 30, reps: int = 5) -> dict:
    """Measured pinned-host <-> device copy rate (best of `reps` 1 GiB copies per
    direction, CUDA events): the PCIe roofline the host-sink copies are quoted against."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for name, dst, src in (("d2h_gbs", h, d), ("h2d_gbs", d, h)):
        best = 0.0
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            e1.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = best
    out["spec_gbs_per_dir"] = 64.0
    log(f"pcie measured: d2h {out['d2h_gbs']:.1f} GB/s h2d {out['h2d_gbs']:.1f} GB/s")
    del h, d
    return out


# ------------------------------------------------------------------ BASELINE.json configs c1, c2, c3, c5
def run_configs(a, ctx, log, peak):
    """Per-config GPU numbers (kc_* calls, CUDA events, L2 flushed) beside the oracle's
    CPU rates on a bounded sample of each config's bytes (bench_configs.py)."""
    import torch
    import bench_configs as bc
    import synth
    timer = bc.Timer(torch, a.config_iters)
    image = open(synth.FIXTURE_CUBIN, "rb").read()
    osec = a.config_oracle_seconds
    out = {}
    t_all = time.perf_counter()

    def fill_c1(vas):
        for spec, arr in zip(synth.C1_SPECS, synth.c1_fill(vas["nodes"])):
            synth.dev_view(vas[spec.name], arr.size).copy_(torch.from_numpy(arr))
    res, pairs, live = bc.closure(
        torch, ctx, timer, synth.C1_SPECS, fill_c1,
        lambda v: dict(image=image, mangled="kc_fixture_walk", grid=(32, 1, 1), block=(256, 1, 1),
                       kernarg=synth.c1_kernarg(v["heads"], v["out"], v["nodes"])), "c1", peak, outputs=("out",))
    res["oracle"] = bc.oracle_both(bc.sample_pairs(torch, [(b, b, n, DTC[d]) for b, _, n, d in pairs], 1 << 20), osec)
    live.release()
    out["c1"] = res
    c2s = synth.c2_specs()

    def fill_c2(vas):
        gen = torch.Generator(device="cuda").manual_seed(synth.seed(2))
        for sp in c2s:
            synth.fill_device(synth.dev_view(vas[sp.name], sp.size), sp, gen)
    res, pairs, live = bc.closure(
        torch, ctx, timer, c2s, fill_c2,
        lambda v: dict(image=image, mangled="kc_fixture_decode_attn", grid=(32, 1, 1), block=(128, 1, 1),
                       kernarg=synth.c2_kernarg(v)), "c2", peak, host=True, outputs=("attn_out",))
    res["oracle"] = bc.oracle_both(bc.sample_pairs(torch, [(b, b, n, DTC[d]) for b, _, n, d in pairs], 64 << 20),
                                   osec)
    live.release()
    out["c2"] = res
    for kind in ("f16", "bf16"):
        res, pairs, keep = bc.c3(torch, ctx, timer, kind, peak)
        res["oracle"] = bc.oracle_both(bc.sample_pairs(torch, pairs[3:] + pairs[:3], 64 << 20), osec)
        del keep
        torch.cuda.empty_cache()
        out[f"c3_{kind}"] = res
    cells = []
    g = torch.Generator(device="cuda").manual_seed(synth.seed(5))
    for S, n in bc.C5_BENCH_CELLS:
        res, pairs, keep = bc.c5_cell(torch, ctx, timer, S, n, peak, g)
        res["oracle_all_cores"] = bc.oracle_rates(bc.sample_pairs(torch, pairs, 32 << 20), os.cpu_count() or 1,
                                                  osec / 2)
        del keep
        torch.cuda.empty_cache()
        cells.append(res)
    out["c5"] = cells
    out["method"] = (f"GPU: CUDA events around each kc_* call, best of {a.config_iters} after one warm-up call, "
                     "L2 flushed before each (512 MiB write, then 512 MiB read: no input line and no dirty line left in L2); closure stages wall-clock around each call. Oracle: "
                     "oracle/ as it stands on a bounded sample of the config's bytes copied back from the device, "
                     "1 thread (first 32 MiB) and every host core")
    out["seconds"] = time.perf_counter() - t_all
    k = out
    log("configs: c2 K1 {:.0f} GB/s ({:.2f}); c3 f16 K2 {:.0f} GB/s ({:.2f}), bf16 K2 {:.0f} GB/s ({:.2f}); "
        "{:.1f} s".format(k["c2"]["K1"]["gbs"], k["c2"]["K1"]["frac"], k["c3_f16"]["K2"]["gbs"],
                          k["c3_f16"]["K2"]["frac"], k["c3_bf16"]["K2"]["gbs"], k["c3_bf16"]["K2"]["frac"],
                          out["seconds"]))
    return out


# oracle dtype codes by the synth dtype names (the kc_dtype numbering)
DTC = {"bytes": 0, "u8": 1, "i8": 2, "u16": 3, "i16": 4, "u32": 5, "i32": 6, "u64": 7, "i64": 8, "f16": 9,
       "bf16": 10, "f32": 11, "f64": 12}


# ------------------------------------------------------------------ oracle (CPU baseline / reference arm)
def c4_sample(pool_or_none, sample_mb: int):
    """A bounded, stratified sample of the c4 workload: the head (whole 64 KiB chunks) of
    EVERY region, sized so the sample is about sample_mb, as (ref, act, dtype) host pairs.
    With a pool: this run's reference bytes copied back (the pool pair is bit-identical,
    so act = ref).  Without (the reference arm, no GPU): regenerated on the host with the
    c4 recipes (bf16 N(0, 0.02) experts, bf16 misc, 10% zero misc, u64 pointer tables)."""
    import numpy as np
    import synth
    specs = synth.c4_specs()
    per = max(65536, (sample_mb * 2**20 // len(specs)) // 65536 * 65536)
    rng = np.random.default_rng(synth.seed(4, 999))
    out = []
    for s in specs:
        k = min(s.size, per)
        if pool_or_none is not None and s.name in pool_or_none.ref:
            v = synth.dev_view(pool_or_none.ref[s.name], k).cpu().numpy().copy()
        elif s.fill == "zero":
            v = np.zeros(k, dtype=np.uint8)
        elif s.fill in ("ptr_table", "topk"):
            v = rng.integers(0, 2**63, size=k // 8, dtype=np.uint64).view(np.uint8)
        else:
            std = s.params.get("std", 1.0)
            v = ((rng.standard_normal(k // 2).astype(np.float32) * np.float32(std)).view(np.uint32) >> 16)
            v = v.astype(np.uint16).view(np.uint8)
        out.append((v, v.copy(), DTC.get(s.dtype, 0)))
    return out


def run_reference(a, rank, world):
    """The reference arm: the CPU oracle as it stands, on every host core, timing the
    metric's step mix (2 manifests of N + the O4 diff reading 2N) over a bounded sample
    of the c4 workload per step; same config/metric/unit as our arm."""
    if rank != 0:
        return None
    import bench_configs as bc
    threads = os.cpu_count() or 1
    sample = c4_sample(None, a.cpu_sample_mb)
    nb = sum(v.size for v, _, _ in sample)
    for _ in range(min(a.warmup, 1)):
        bc.oracle_rates(sample[:4], threads, 0.0)
    steps = []
    for _ in range(a.steps):
        r = bc.oracle_rates(sample, threads, a.ref_step_seconds / 2)
        steps.append(r)
    secs = sum(r["hash_s"] + r["diff_s"] for r in steps)
    value = sum(r["step_mix_gbs"] for r in steps) / len(steps)
    desc = (f"the first {nb // 185 // 1024} KiB of every one of the 185 c4 regions ({nb / 1e6:.1f} MB, regenerated "
            f"on the host with the c4 recipes); per step: O2 manifests repeated >= {a.ref_step_seconds / 2:.1f} s, "
            f"the O4 diff repeated >= {a.ref_step_seconds / 2:.1f} s; value = 4N / (2N/hash + 2N/diff)")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * secs / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic", "config": workload_config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc,
                             "hash_gbs": sum(r["hash_gbs"] for r in steps) / len(steps),
                             "diff_gbs": sum(r["diff_gbs"] for r in steps) / len(steps),
                             "host": bc.host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-fused", action="store_true", help="skip the F2 fused-step measurement")
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--cpu-sample-mb", type=int, default=384)
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--ref-step-seconds", type=float, default=5.0)
    p.add_argument("--no-latency", action="store_true")
    p.add_argument("--latency-dir", default="/dev/shm/kc_bench_capture")
    p.add_argument("--quiet", action="store_true")
    p.add_argument("--plant", action="store_true",
                   help="plant 1-byte mismatches in the reference pool (deterministic by region, so the N-GPU "
                        "reports and bitmaps can be compared with the 1-GPU ones); never a headline number")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-configs", action="store_true", help="skip the c1/c2/c3/c5 per-config measurements")
    p.add_argument("--config-iters", type=int, default=5)
    p.add_argument("--config-oracle-seconds", type=float, default=1.0)
    p.add_argument("--combine", default="nccl", choices=["nccl", "peer"],
                   help="N > 1, E1: nccl = C2/C3/C4 collectives; peer = K1/K2 write the post-manifest, reports "
                        "and bitmaps straight into rank 0's HBM through peer mappings, the exchange a barrier")
    p.add_argument("--placement", default="e1", choices=["e1", "e2"],
                   help="e1: residency-first shards (each rank reads its own HBM; the headline); e2: the pool "
                        "resident on rank 0, every rank reading a 1/N share of it over NVLink peer mappings "
                        "(bounded by rank 0's HBM, SURVEY.md 8(e))")
    p.add_argument("--replay-child", default=None, help=argparse.SUPPRESS)
    a = p.parse_args()
    if a.replay_child:
        replay_child(a.replay_child)
        return
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        # one process per GPU: launch the ranks ourselves (the driver's torchrun line,
        # run from here), rendezvous on 127.0.0.1; rank 0 prints the JSON line
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        print(json.dumps({"error": f"--gpus {a.gpus} but WORLD_SIZE {world}: launch one rank per GPU"}), flush=True)
        sys.exit(2)
    log = (lambda m: None) if a.quiet else (lambda m: print(m, file=sys.stderr, flush=True))

    if a.impl == "reference":
        res = run_reference(a, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    # KC_BENCH_ONE_GPU=1 + KC_BENCH_BACKEND=gloo: every rank on cuda:0, collectives through
    # host memory -- a functional check of the N > 1 path on a single-GPU box, never a number
    device = 0 if os.environ.get("KC_BENCH_ONE_GPU") else local
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(device)
        backend = os.environ.get("KC_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{device}"))
        else:
            dist.init_process_group(backend)
    if world == 1:
        a.placement = "e1"   # one rank: the pool is resident and local either way
    res, pool = run_ours(a, rank, world, device, log)
    if world > 1:
        res["collectives"] = {"backend": torch.distributed.get_backend(),
                                        "nccl": ".".join(map(str, torch.cuda.nccl.version())),
                                        "step": ("peer combine: K1's post-manifest, K2's reports and bitmaps "
                                                 "written into rank 0's HBM through peer mappings, then a barrier"
                                                 if a.combine == "peer" and a.placement == "e1" else
                                                 "C2 all_gather manifests, C3 all_reduce SUM/MAX reports, "
                                                 "C4 all_gather per-region bitmaps")}
    if os.environ.get("KC_BENCH_ONE_GPU") and world > 1:
        res["functional_check_only"] = "all ranks on cuda:0 (KC_BENCH_ONE_GPU)"
    if a.plant:
        res["planted"] = "reference pool planted with 1-byte mismatches (--plant): a parity run"
    if rank == 0 and world == 1 and not a.no_configs:
        res["configs"] = run_configs(a, pool.ctx, log, res["roofline"]["peak"])
    if rank == 0 and world == 1 and not a.no_cpu_baseline:   # the oracle baseline: rank 0 at N = 1 only
        import bench_configs as bc
        threads = os.cpu_count() or 1
        sample = c4_sample(pool, a.cpu_sample_mb)
        nb = sum(v.size for v, _, _ in sample)
        rates = bc.oracle_both(sample, a.cpu_seconds / 4, threads)
        res["cpu_baseline"] = {"value": rates["all_cores"]["step_mix_gbs"], "unit": UNIT, "cores": threads,
                               "kind": "oracle",
                               "sample": f"this run's c4 pool: the first {nb // 185 // 1024} KiB of every one of "
                                         f"the 185 regions ({nb / 1e6:.1f} MB, copied back from HBM); O2 manifests "
                                         f"and the O4 diff each repeated >= {a.cpu_seconds / 4:.1f} s at 1 thread "
                                         f"(first 32 MiB) and at {threads} threads; value = the metric's step mix "
                                         f"4N / (2N/hash + 2N/diff) at {threads} threads",
                               "hash_gbs": {"t1": rates["t1"]["hash_gbs"], "all_cores": rates["all_cores"]["hash_gbs"]},
                               "diff_gbs": {"t1": rates["t1"]["diff_gbs"], "all_cores": rates["all_cores"]["diff_gbs"]},
                               "step_mix_gbs_t1": rates["t1"]["step_mix_gbs"], "host": bc.host_info()}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
