"""A9 combine logic at world size 2 over gloo on CPU (O7: N-GPU == 1-GPU bit for bit).

Each rank owns a residency-first share of a synthetic heap; its local manifests
and reports come from the oracle (standing in for its GPU's K1/K2 output), the
product's combine functions (paper_2605_03208_b200.dist) merge them, and the
result must equal the oracle run over the whole heap on one process.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

CH = 65536


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _heap():
    rng = np.random.default_rng(42)
    sizes = [3 * CH + 5, 64 * CH, 17, 5 * CH, 2 * CH - 1, 130 * CH + 33]
    bases = [0x7F0000000000 + i * (256 << 20) for i in range(len(sizes))][::-1]  # unsorted on purpose
    data = [rng.integers(0, 256, size=n, dtype=np.uint8) for n in sizes]
    owner = [i % 2 for i in range(len(sizes))]
    return bases, sizes, owner, data


def _worker(rank, world, port, errq):
    try:
        import torch.distributed as dist
        import oracle
        from paper_2605_03208_b200 import dist as kd
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        bases, sizes, owner, data = _heap()
        plan = kd.Plan.from_rank0(bases if rank == 0 else None, sizes if rank == 0 else None,
                                  owner if rank == 0 else None) if rank == 0 else kd.Plan.from_rank0(None, None, None)
        # ---- C2: manifests
        by_base = {b: d for b, d in zip(bases, data)}
        local = [oracle.chunk_hashes(by_base[b]) for b, _ in plan.local_regions()]
        local_h = torch.from_numpy(np.concatenate(local).view(np.int64)) if local else torch.zeros(0, dtype=torch.int64)
        got = plan.gather_manifest(local_h).numpy().view(np.uint64)
        order = sorted(range(len(bases)), key=lambda i: bases[i])
        whole = np.concatenate([oracle.chunk_hashes(data[i]) for i in order])
        assert np.array_equal(got, whole), "gathered manifest != 1-process manifest"

        # ---- C4 per-region bitmaps (E1: each region on one rank): gathered in global order
        def act_of(b, d):
            a = d.copy()
            a[(b >> 20) % d.size] ^= 0x10                  # one flipped byte per region, VA-seeded
            if d.size > 70 * CH:
                a[66 * CH + 3] ^= 1
            return a
        lw = [oracle.diff(by_base[b], act_of(b, by_base[b])).bitmap for b, _ in plan.local_regions()]
        local_w = torch.from_numpy(np.concatenate(lw).view(np.int64)) if lw else torch.zeros(0, dtype=torch.int64)
        got_bm = kd.gather_region_bitmaps(plan, local_w).numpy().view(np.uint64)
        whole_bm = np.concatenate([oracle.diff(data[i], act_of(bases[i], data[i])).bitmap for i in order])
        assert np.array_equal(got_bm, whole_bm), "gathered per-region bitmaps != 1-process bitmaps"

        # ---- C3/C4 on a buffer split across the ranks (chunk-aligned halves)
        rng = np.random.default_rng(7)
        n_el = 2 * (128 * CH) // 2  # bf16 elements of a 2 x 4 MiB buffer
        ref = (rng.standard_normal(n_el).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        act = ref.copy()
        m = rng.random(n_el) < 0.05
        act[m] ^= 1
        act[10] = 0x7FC1                                   # NaN in A
        ref[n_el - 3] = 0; act[n_el - 3] = 1               # rel undefined, in rank 1's half
        rb, ab = ref.view(np.uint8), act.view(np.uint8)
        half = rb.size // 2
        lo, hi = rank * half, (rank + 1) * half
        loc = oracle.diff(rb[lo:hi], ab[lo:hi], oracle.DT_BF16)
        row = np.zeros(15, dtype=np.int64)
        r = loc.report
        row[kd.DIFF_BYTES] = r["differing_bytes"]; row[kd.DIFF_ELEMS] = r["differing_elems"]
        row[kd.MAX_ULP] = np.int64(np.uint64(r["max_ulp"]).view(np.int64))
        row[kd.MAX_ABS] = np.array([r["max_abs"]]).view(np.int64)[0]
        row[kd.MAX_REL] = np.array([r["max_rel"]]).view(np.int64)[0]
        row[kd.NAN_REF] = r["nan_ref"]; row[kd.NAN_ACT] = r["nan_act"]; row[kd.NAN_POS] = r["nan_pos_mismatch"]
        row[kd.REL_UNDEF] = r["rel_undefined"]; row[kd.ALLCLOSE_FAIL] = r["allclose_fail"]
        comb = kd.combine_reports(torch.from_numpy(row).view(1, 15))
        fin = kd.finalize(comb, [rb.size], ["bf16"])[0]
        exp = oracle.diff(rb, ab, oracle.DT_BF16)
        for k, v in exp.report.items():
            assert fin[k] == v, f"{k}: combined {fin[k]} != whole {v}"
        nwords = (rb.size // CH + 63) // 64
        words = np.zeros(nwords, dtype=np.uint64)
        lb = loc.bitmap
        c0 = lo // CH
        for k in range(half // CH):
            if (int(lb[k // 64]) >> (k % 64)) & 1:
                g = c0 + k
                words[g // 64] |= np.uint64(1) << np.uint64(g % 64)
        gb = kd.gather_bitmaps(torch.from_numpy(words.view(np.int64))).numpy().view(np.uint64)
        assert np.array_equal(gb, exp.bitmap), "combined bitmap != whole bitmap"

        # ---- max_ulp above 2^63 survives the signed MAX (f64 -inf vs +inf)
        big = torch.zeros(1, 15, dtype=torch.int64)
        if rank == 1:
            big[0, kd.MAX_ULP] = np.int64(np.uint64(0xFFE0000000000000).view(np.int64))
        else:
            big[0, kd.MAX_ULP] = 5
        c = kd.combine_reports(big)
        assert (int(c[0, kd.MAX_ULP]) & 0xFFFFFFFFFFFFFFFF) == 0xFFE0000000000000
        dist.destroy_process_group()
    except Exception as e:  # surface to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


@pytest.mark.timeout(300)
def test_combine_world2_gloo_equals_single_process():
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs)


def test_plan_permutation_single_rank_is_identity():
    from paper_2605_03208_b200.dist import Plan
    p = Plan([0, 1 << 30, 2 << 30], [CH * 3, 5, CH], [0, 0, 0], 1, 0)
    assert p.manifest_permutation().tolist() == list(range(p.global_chunks()))
    p2 = Plan([0, 1 << 30, 2 << 30], [CH * 3, 5, CH], [1, 0, 1], 2, 0)
    # rank 0 holds region 1 (1 chunk), rank 1 holds regions 0 and 2 (3 + 1 chunks); pad = 4
    assert p2.manifest_permutation().tolist() == [4, 5, 6, 0, 7]


def test_plan_bitmap_permutation():
    from paper_2605_03208_b200.dist import Plan
    # sizes: 130 chunks (3 words), 1 chunk (1 word), 64 chunks (1 word); owners 1, 0, 1
    p = Plan([0, 1 << 30, 2 << 30], [CH * 130, 5, CH * 64], [1, 0, 1], 2, 0)
    # rank 0 words: [r1]; rank 1 words: [r0 x3, r2]; pad = 4
    assert p.bitmap_words(0) == 1 and p.bitmap_words(1) == 4
    assert p.bitmap_permutation().tolist() == [4, 5, 6, 0, 7]


def test_report_finalize_in_the_library_matches_the_oracle_rules():
    """kc_report_finalize (host, no CUDA) on counters the oracle produced: the derived
    fields equal the oracle's own report (1 of 1024 bytes -> 0.09765625)."""
    import oracle
    from paper_2605_03208_b200 import kc
    ref = np.zeros(1024, dtype=np.uint8)
    act = ref.copy()
    act[5] = 1
    for dt, name in ((oracle.DT_BYTES, "bytes"), (oracle.DT_U32, "u32"), (oracle.DT_F32, "f32")):
        exp = oracle.diff(ref, act, dt).report
        row = np.zeros(15, dtype=np.int64)
        row[3], row[4], row[5] = exp["differing_bytes"], exp["differing_elems"], exp["max_ulp"]
        row[9:14] = [exp[k] for k in ("nan_ref", "nan_act", "nan_pos_mismatch", "rel_undefined", "allclose_fail")]
        row[6] = np.array([exp["max_abs"]]).view(np.int64)[0]
        row[7] = np.array([exp["max_rel"]]).view(np.int64)[0]
        got = kc.report_finalize(row.reshape(1, 15), [1024], [name])[0]
        assert got == exp, (name, got, exp)
        assert got["percent_bytes"] == 0.09765625
    with pytest.raises(kc.KcError):
        kc.report_finalize(np.zeros((1, 15), dtype=np.int64), [1023], ["u32"])
