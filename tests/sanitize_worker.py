"""Workload for the compute-sanitizer runs (tests/test_gpu_sanitizer.py,
SURVEY.md §5 "Race detection / sanitizers"): every kernel of the path at small
sizes, each result checked against the oracle so a sanitizer-clean run is also a
correct one.

  K1 cp.async ring, both configurations: CpS (sub-wave snapshots) and CpA (>= 148 x 8
     groups, 640 MiB, so CTAs loop over their rings), plus the unaligned generic path;
  K3 written set; digest kernels;
  K2 every dtype family, planted mismatches and Inf/NaN, ragged tails, misaligned bases;
  K5 + filtered K2 (kc_hash_diff_async);
  K6 fused capture (hash + copy into the arena) and the fused restore, K4 gather, replay
     and validate: the c1 closure through __graft_entry__.smoke() and a 640 MiB capture.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tests/sanitize_worker.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path[:0] = [ROOT, HERE]
CH = 65536


def main():
    import torch

    import __graft_entry__
    import oracle
    import synth
    from paper_2605_03208_b200 import kc
    from test_gpu_diff import _dev, _pair_host, _same

    __graft_entry__.smoke()          # K1, K3, K2, digests; c1 capture (K6) -> restore -> replay -> validate
    torch.cuda.set_device(0)
    ctx = kc.Context(0)
    u64 = lambda t: t.cpu().numpy().view(np.uint64)

    # K1 CpA (the large-snapshot ring) + ragged CpS tails in one call
    g = torch.Generator(device="cuda").manual_seed(5)
    big = torch.randint(0, 256, (640 * 2**20 + 4096 + 24,), dtype=torch.uint8, device="cuda", generator=g)
    small = torch.randint(0, 256, (3 * CH + 40,), dtype=torch.uint8, device="cuda", generator=g)
    bufs = sorted([big, small], key=lambda t: t.data_ptr())
    regions = [(b.data_ptr(), b.numel()) for b in bufs]
    C = kc.count_chunks(regions)
    assert (C + 7) // 8 >= 148 * 8
    h = torch.zeros(C, dtype=torch.int64, device="cuda")
    ctx.hash(regions, h.data_ptr())
    torch.cuda.synchronize()
    exp = np.concatenate([oracle.chunk_hashes(b.cpu().numpy()) for b in bufs])
    assert np.array_equal(u64(h), exp), "K1 CpA != oracle"
    h2 = torch.zeros(kc.count_chunks([(small.data_ptr() + 3, 2 * CH + 5)]), dtype=torch.int64, device="cuda")
    ctx.hash([(small.data_ptr() + 3, 2 * CH + 5)], h2.data_ptr())    # unaligned base: generic path
    torch.cuda.synchronize()
    assert np.array_equal(u64(h2), oracle.chunk_hashes(small.cpu().numpy()[3:3 + 2 * CH + 5])), "K1 generic"
    print("K1 CpA/CpS/generic ok", flush=True)

    # K2, every dtype family, planted mismatches and specials; one misaligned pair
    for dtname in ["bytes", "u8", "i16", "u32", "i64", "f16", "bf16", "f32", "f64"]:
        dt = oracle.DTYPE_NAMES.index(dtname)
        s = oracle.ELEM_SIZE[dt]
        for nbytes, off in [(3 * CH + 40, (0, 0)), (700 * 1024 + 24, (0, 0)), (8, (0, 0)), (2 * CH + 96, (s, 3 * s))]:
            r, a = _pair_host(dt, nbytes // s, seed=nbytes + dt, orc=oracle)
            tr, pr = _dev(torch, r, off[0])
            ta, pa = _dev(torch, a, off[1])
            reps, bms = ctx.diff([(pr, pa, r.size, dtname)])
            e = oracle.diff(r, a, dt)
            _same(reps[0], e.report, f"K2 {dtname} {nbytes}")
            assert [int(w) for w in bms[0]] == [int(w) for w in e.bitmap], f"K2 bitmap {dtname}"
    print("K2 ok", flush=True)

    # K5 fused hash + compare, then K2 over the dirty chunks only
    pairs = []
    for j, dtname in enumerate(["bf16", "f32", "bytes", "f16"]):
        dt = oracle.DTYPE_NAMES.index(dtname)
        s = oracle.ELEM_SIZE[dt]
        n = (5 + 7 * j) * CH + 32 * j
        r, a = _pair_host(dt, n // s, seed=40 + j, orc=oracle, specials=j == 0, density=0.113 if j % 2 == 0 else 1e-5)
        pairs.append((dtname, r, a))
    keep, kb = [], []
    for dtname, r, a in pairs:
        tr, pr = _dev(torch, r)
        ta, pa = _dev(torch, a)
        keep += [tr, ta]
        kb.append((pr, pa, r.size, dtname))
    nch = [(r.size + CH - 1) // CH for _, r, _ in pairs]
    words = [(c + 63) // 64 for c in nch]
    d_h = torch.zeros(sum(nch), dtype=torch.int64, device="cuda")
    d_rep = torch.zeros(len(pairs) * 15, dtype=torch.int64, device="cuda")
    d_bm = torch.zeros(sum(words), dtype=torch.int64, device="cuda")
    d_dirty = torch.zeros((sum(nch) + 63) // 64, dtype=torch.int64, device="cuda")
    ctx.hash_diff_async(kb, d_h.data_ptr(), d_rep.data_ptr(), d_bm.data_ptr(), d_dirty.data_ptr())
    torch.cuda.synchronize()
    raw, bm = d_rep.cpu().numpy().tobytes(), u64(d_bm)
    c0 = w0 = 0
    for j, (dtname, r, a) in enumerate(pairs):
        dt = oracle.DTYPE_NAMES.index(dtname)
        assert np.array_equal(u64(d_h)[c0:c0 + nch[j]], oracle.chunk_hashes(a)), f"K5 manifest {dtname}"
        e = oracle.diff(r, a, dt)
        _same(kc.DiffReport.from_buffer_copy(raw[120 * j:120 * (j + 1)]).as_dict(), e.report, f"K5+K2 {dtname}")
        assert [int(x) for x in bm[w0:w0 + words[j]]] == [int(x) for x in e.bitmap]
        c0, w0 = c0 + nch[j], w0 + words[j]
    print("K5 + filtered K2 ok", flush=True)

    # prepared plans (K1 / K2 from plan-owned tables) and the byte-exact host-reference
    # validation (staging ring on the copy stream, K2 accumulating over pieces)
    hp = ctx.hash_plan(regions)
    hp.run(h.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(u64(h), exp), "K1 plan != oracle"
    hp.close()
    nbs = [r.size for _, r, _ in pairs]
    w0s = list(np.cumsum([0] + words[:-1]))
    dp = ctx.diff_plan(kb, len(kb), nbs, w0s)
    dp.run(d_rep.data_ptr(), d_bm.data_ptr())
    torch.cuda.synchronize()
    raw = d_rep.cpu().numpy().tobytes()
    for j, (dtname, r, a) in enumerate(pairs):
        e = oracle.diff(r, a, oracle.DTYPE_NAMES.index(dtname))
        _same(kc.DiffReport.from_buffer_copy(raw[120 * j:120 * (j + 1)]).as_dict(), e.report, f"K2 plan {dtname}")
    dp.close()
    hostb, hb = [], []
    for (dtname, r, a), (pr, pa, nb, _) in zip(pairs, kb):
        hr = torch.from_numpy(r).pin_memory()
        hostb.append(hr)
        hb.append((hr.data_ptr(), pa, nb, dtname))
    reps, bms, moved = ctx.validate_host_ref(hb, 0)
    assert moved == sum(nbs)
    for j, (dtname, r, a) in enumerate(pairs):
        _same(reps[j], oracle.diff(r, a, oracle.DTYPE_NAMES.index(dtname)).report, f"byte-exact host ref {dtname}")
    print("plans + byte-exact host-reference validation ok", flush=True)

    # K6 on the CpA ring: a 640 MiB region next to the c1 closure, captured into HBM,
    # restored at the same VAs (fused restore), replayed and validated
    sizes = [s.size for s in synth.C1_SPECS] + [640 * 2**20]
    vas = [ctx.alloc(sz) for sz in sizes]
    nodes_va, heads_va, out_va, pad_va = vas
    init = synth.c1_fill(nodes_va)
    for va, arr in zip(vas, init):
        synth.dev_view(va, arr.size).copy_(torch.from_numpy(arr))
    synth.dev_view(pad_va, sizes[3]).copy_(big[:sizes[3]])
    torch.cuda.synchronize()
    for mode in (kc.KC_MODE_PRE_W, kc.KC_MODE_POST):
        snap, _ = ctx.capture_dev(image=open(synth.FIXTURE_CUBIN, "rb").read(), mangled="kc_fixture_walk",
                                  grid=(32, 1, 1), block=(256, 1, 1), mode=mode,
                                  kernarg=synth.c1_kernarg(heads_va, out_va, nodes_va, mutate=1))
        post = {va: synth.dev_view(va, sz).cpu().numpy().copy() for va, sz in zip(vas, sizes)}
        for va in vas:
            ctx.free(va)
        r, _ = ctx.restore_dev(snap)
        if mode == kc.KC_MODE_PRE_W:
            ctx.replay(r)
        reps, unexpected = ctx.validate(r)
        assert reps and all(x["differing_bytes"] == 0 for x in reps) and unexpected == 0, f"K6 closure mode {mode}"
        for va, sz in zip(vas, sizes):
            assert np.array_equal(synth.dev_view(va, sz).cpu().numpy(), post[va]), f"restored state mode {mode}"
        r.release()
        snap.free()
        vas = [ctx.alloc(sz) for sz in sizes]
        nodes_va, heads_va, out_va, pad_va = vas
        init = synth.c1_fill(nodes_va)
        for va, arr in zip(vas, init):
            synth.dev_view(va, arr.size).copy_(torch.from_numpy(arr))
        synth.dev_view(pad_va, sizes[3]).copy_(big[:sizes[3]])
        torch.cuda.synchronize()
    for va in vas:
        ctx.free(va)
    print("K6 capture / fused restore / replay / validate ok", flush=True)
    ctx.close()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
