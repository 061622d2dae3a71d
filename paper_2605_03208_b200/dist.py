"""A9: multi-GPU combine of manifests and diff reports over torch.distributed.

SURVEY.md 8(e): chunks are independent for K1 and K2 and every combine is a
concatenation, a SUM or a MAX, so the N-GPU result equals the 1-GPU result bit
for bit (O7).  Placement is residency-first (E1): each rank hashes/diffs the
regions resident in its own HBM.  Collectives (NCCL on GPUs, gloo on CPU):

  C1  broadcast of the global region table + owner map (Plan.from_rank0)
  C2  all_gather of per-rank chunk manifests, reordered into global chunk order
  C3  all_reduce SUM of report counters and MAX of report maxima
  C4  all_gather (bitwise OR) of mismatch-bitmap words

Host logic only: every byte of hashing and diffing happened in libkc.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

CHUNK = 65536
REP_WORDS = 15  # sizeof(kc_diff_report) / 8
# kc_diff_report word offsets (include/kc.h)
NBYTES, N_ELEMS, N_CHUNKS, DIFF_BYTES, DIFF_ELEMS, MAX_ULP, MAX_ABS, MAX_REL, PERCENT = range(9)
NAN_REF, NAN_ACT, NAN_POS, REL_UNDEF, ALLCLOSE_FAIL, PASS = range(9, 15)
SUM_FIELDS = [DIFF_BYTES, DIFF_ELEMS, NAN_REF, NAN_ACT, NAN_POS, REL_UNDEF, ALLCLOSE_FAIL]
MAX_FIELDS = [MAX_ULP, MAX_ABS, MAX_REL]
_SIGN = -(1 << 63)


def _nchunks(size: int) -> int:
    return (size + CHUNK - 1) // CHUNK


def _bitmap_words(size: int) -> int:
    return (_nchunks(size) + 63) // 64


def _host_staged(group) -> bool:
    """gloo cannot run these collectives on CUDA tensors: stage through host memory."""
    return dist.get_backend(group) == "gloo"


def _all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None) -> None:
    if _host_staged(group) and inp.is_cuda:
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def _all_reduce(t: torch.Tensor, op, group=None) -> None:
    if _host_staged(group) and t.is_cuda:
        c = t.cpu()
        dist.all_reduce(c, op=op, group=group)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op, group=group)


@dataclass
class Plan:
    """Global region table (sorted by base) with the owning rank of each region."""
    bases: list
    sizes: list
    owner: list
    world: int
    rank: int

    @staticmethod
    def from_rank0(bases, sizes, owner, group=None, device="cpu") -> "Plan":
        """C1: rank 0's table is broadcast to every rank (other ranks may pass None)."""
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        if _host_staged(group):
            device = "cpu"
        n = torch.tensor([len(bases) if rank == 0 else 0], dtype=torch.int64, device=device)
        dist.broadcast(n, 0, group=group)
        t = torch.zeros(3, int(n.item()), dtype=torch.int64, device=device)
        if rank == 0:
            t[0] = torch.tensor(list(bases), dtype=torch.int64)
            t[1] = torch.tensor(list(sizes), dtype=torch.int64)
            t[2] = torch.tensor(list(owner), dtype=torch.int64)
        dist.broadcast(t, 0, group=group)
        order = torch.argsort(t[0].cpu(), stable=True)
        tc = t.cpu()[:, order]
        return Plan(tc[0].tolist(), tc[1].tolist(), tc[2].tolist(), world, rank)

    # -- per-rank views
    def local_regions(self, r=None):
        r = self.rank if r is None else r
        return [(b, s) for b, s, o in zip(self.bases, self.sizes, self.owner) if o == r]

    def local_chunks(self, r=None) -> int:
        return sum(_nchunks(s) for _, s in self.local_regions(r))

    def max_local_chunks(self) -> int:
        return max(self.local_chunks(r) for r in range(self.world))

    def global_chunks(self) -> int:
        return sum(_nchunks(s) for s in self.sizes)

    def bitmap_words(self, r=None) -> int:
        """Bitmap words of rank r's regions (one ceil(n_chunks/64)-word bitmap per region)."""
        return sum(_bitmap_words(s) for _, s in self.local_regions(r))

    def bitmap_permutation(self) -> torch.Tensor:
        """Index into the gathered [world, max_local_words] bitmap words that yields
        every region's bitmap in global (ascending base) order."""
        pad = max(1, max(self.bitmap_words(r) for r in range(self.world)))
        offs = [0] * self.world
        idx = []
        for s, o in zip(self.sizes, self.owner):
            n = _bitmap_words(s)
            idx.extend(range(o * pad + offs[o], o * pad + offs[o] + n))
            offs[o] += n
        return torch.tensor(idx, dtype=torch.int64)

    def manifest_permutation(self) -> torch.Tensor:
        """Index into the gathered [world, max_local] manifest that yields global chunk order."""
        pad = self.max_local_chunks()
        offs = [0] * self.world
        idx = []
        for s, o in zip(self.sizes, self.owner):
            n = _nchunks(s)
            idx.extend(range(o * pad + offs[o], o * pad + offs[o] + n))
            offs[o] += n
        return torch.tensor(idx, dtype=torch.int64)

    # -- C2
    def gather_manifest(self, local_h: torch.Tensor, perm: torch.Tensor | None = None, group=None) -> torch.Tensor:
        """All-gather the per-rank manifests (int64 views of the u64 hashes, local
        regions in ascending base) and return the global manifest."""
        pad = self.max_local_chunks()
        mine = torch.zeros(max(1, pad), dtype=torch.int64, device=local_h.device)
        n = self.local_chunks()
        mine[:n].copy_(local_h[:n])
        out = torch.empty(self.world * max(1, pad), dtype=torch.int64, device=local_h.device)
        _all_gather_into(out, mine, group)
        if perm is None:
            perm = self.manifest_permutation()
        return out.index_select(0, perm.to(local_h.device))


# ------------------------------------------------------------------ C3
def combine_reports(reps: torch.Tensor, group=None) -> torch.Tensor:
    """All-reduce per-buffer reports ([R, 15] int64 view of kc_diff_report):
    SUM of the counters, MAX of max_ulp (unsigned, order-preserving sign flip)
    and of max_abs / max_rel (non-negative doubles order like their bits).
    nbytes/n_elems/n_chunks/percent/pass are recomputed by :func:`finalize`."""
    out = reps.clone()
    s = reps[:, SUM_FIELDS].contiguous()
    _all_reduce(s, dist.ReduceOp.SUM, group)
    m = reps[:, MAX_FIELDS].contiguous()
    m[:, 0] ^= _SIGN
    _all_reduce(m, dist.ReduceOp.MAX, group)
    m[:, 0] ^= _SIGN
    out[:, SUM_FIELDS] = s
    out[:, MAX_FIELDS] = m
    return out


def finalize(combined: torch.Tensor, nbytes: list, dtypes: list) -> list:
    """Report dicts of a combined report table: the derived fields (n_elems,
    n_chunks, percent_bytes, pass) are recomputed by the library
    (kc_report_finalize, K2's finalize rules), not here."""
    from . import kc
    return kc.report_finalize(combined.cpu().numpy(), nbytes, dtypes)


# ------------------------------------------------------------------ C4
def gather_bitmaps(local_words: torch.Tensor, group=None) -> torch.Tensor:
    """Bitwise OR of every rank's bitmap words (ranks hold disjoint chunks under
    E1, so the OR is a concatenation; split buffers OR their bits)."""
    world = dist.get_world_size(group)
    out = torch.empty(world * local_words.numel(), dtype=local_words.dtype, device=local_words.device)
    _all_gather_into(out, local_words.contiguous(), group)
    acc = out.view(world, -1)[0].clone()
    for r in range(1, world):
        acc |= out.view(world, -1)[r]
    return acc


def gather_region_bitmaps(plan: Plan, local_words: torch.Tensor, perm: torch.Tensor | None = None,
                          group=None) -> torch.Tensor:
    """C4 for per-region bitmaps under E1 (each region wholly on one rank): all-gather
    every rank's words (its regions in ascending base, ceil(n_chunks/64) words each)
    and return them in global region order -- the 1-GPU kc_diff bitmap layout."""
    pad = max(1, max(plan.bitmap_words(r) for r in range(plan.world)))
    mine = torch.zeros(pad, dtype=torch.int64, device=local_words.device)
    n = plan.bitmap_words()
    mine[:n].copy_(local_words[:n])
    out = torch.empty(plan.world * pad, dtype=torch.int64, device=local_words.device)
    _all_gather_into(out, mine, group)
    if perm is None:
        perm = plan.bitmap_permutation()
    return out.index_select(0, perm.to(local_words.device))


def gather_ranges(local: torch.Tensor, counts: list, group=None) -> torch.Tensor:
    """C2 under E2 (contiguous chunk ranges per rank, in rank order): all-gather
    the per-rank manifests, padded to the largest count, and concatenate the
    valid prefixes -- the global manifest."""
    world = len(counts)
    pad = max(1, max(counts))
    mine = torch.zeros(pad, dtype=local.dtype, device=local.device)
    r = dist.get_rank(group)
    mine[:counts[r]].copy_(local[:counts[r]])
    out = torch.empty(world * pad, dtype=local.dtype, device=local.device)
    _all_gather_into(out, mine, group)
    return torch.cat([out[i * pad:i * pad + counts[i]] for i in range(world)])
