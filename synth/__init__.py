"""Seeded synthetic inputs for the Kerncap closure hot path.

This module holds NONE of the method's arithmetic (no hashing, no diffing, no
ULP/abs/rel): it only lays out regions and fills them with seeded values in
the shapes, sizes and value distributions of the paper's workloads.  Both the
CUDA path and the oracle consume what it produces (the oracle always reads the
materialised bytes back, it never regenerates them).  Seeds are
260503208 + config number (SURVEY.md:987-988).

Configs (BASELINE.json ``configs``):
  c1  1 MiB heap, 3 allocations incl. a pointer-chasing linked list
  c2  152 MiB llama.cpp-shaped snapshot (21 regions) + decode-attention dispatch
  c3  2 GiB fp16/bf16 attention-forward buffer set with planted ULP-level mismatches
  c4  30,074,000,000 B vLLM-style MoE weight pool (185 regions) reached via pointer tables
  c5  region-size/count sweep
"""
from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 260503208
CHUNK = 65536
FIXTURE_CUBIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "kc_fixtures.cubin")


def seed(cfg: int, stream: int = 0) -> int:
    return SEED_BASE + cfg + 1000 * stream


@dataclass
class RegionSpec:
    """One allocation of a synthetic heap: name, exact size, element type and fill recipe."""
    name: str
    size: int
    dtype: str = "bytes"          # interpretation for typed validation
    fill: str = "zero"            # zero | u8 | u8range | normal | arange_i32 | kv
    params: dict = field(default_factory=dict)
    layer: int = -1               # c4: owning MoE layer (-1 = misc)


# ------------------------------------------------------------------ c1
C1_N_LISTS = 8192
C1_LIST_LEN = 5
C1_N_NODES = C1_N_LISTS * C1_LIST_LEN            # 40,960 x 16 B = 655,360 B
C1_SPECS = [RegionSpec("nodes", 16 * C1_N_NODES), RegionSpec("heads", 8 * C1_N_LISTS),
            RegionSpec("out", 8 * C1_N_NODES, dtype="u64")]


def c1_fill(nodes_va: int, n_lists: int = C1_N_LISTS, list_len: int = C1_LIST_LEN, s: int | None = None):
    """Bytes of (nodes, heads, out) for the c1 linked-list heap.

    Node slots are placed by a seeded random permutation; values uniform u32;
    next pointers are device VAs inside the nodes allocation (T**-style)."""
    rng = np.random.default_rng(seed(1) if s is None else s)
    n_nodes = n_lists * list_len
    slots = rng.permutation(n_nodes).astype(np.uint64)
    values = rng.integers(0, 2**32, size=n_nodes, dtype=np.uint64).astype(np.uint32)
    nodes = np.zeros(n_nodes, dtype=[("next", "<u8"), ("value", "<u4"), ("pad", "<u4")])
    order = slots.reshape(n_lists, list_len)
    nxt = np.zeros((n_lists, list_len), dtype=np.uint64)
    nxt[:, :-1] = np.uint64(nodes_va) + np.uint64(16) * order[:, 1:]
    nodes["next"][order.reshape(-1)] = nxt.reshape(-1)
    nodes["value"][order.reshape(-1)] = values
    heads = (np.uint64(nodes_va) + np.uint64(16) * order[:, 0]).astype(np.uint64)
    out = np.zeros(n_nodes, dtype=np.uint64)
    return np.frombuffer(nodes.tobytes(), dtype=np.uint8).copy(), heads.view(np.uint8).copy(), out.view(np.uint8).copy()


def c1_kernarg(heads_va: int, out_va: int, nodes_va: int, n_lists: int = C1_N_LISTS, mutate: int = 0) -> bytes:
    """Packed parameter buffer of kc_fixture_walk (natural alignment: 8,8,8,4,4)."""
    return struct.pack("<QQQIi", heads_va, out_va, nodes_va, n_lists, mutate)


# ------------------------------------------------------------------ c2
def c2_specs() -> list:
    specs = [RegionSpec(f"w_q{i}", 8 * 2**20, "u8", "u8") for i in range(12)]
    specs += [
        RegionSpec("w_scales", 6 * 2**20, "u8", "u8range", {"lo": 118, "hi": 136}),
        RegionSpec("k_cache", 16 * 2**20, "f16", "kv", {"valid": 3072, "ctx": 4096}),
        RegionSpec("v_cache", 16 * 2**20, "f16", "kv", {"valid": 3072, "ctx": 4096}),
        RegionSpec("q", 2**20, "f16", "normal", {"std": 1.0}),
        RegionSpec("attn_out", 2**20, "f32", "zero"),
        RegionSpec("workspace", 12 * 2**20, "f32", "zero"),
        RegionSpec("pos", 2**20, "i32", "arange_i32"),
        RegionSpec("mask", 2**20, "f16", "zero"),
        RegionSpec("logits", 2 * 2**20, "f32", "normal", {"std": 1.0}),
    ]
    assert sum(s.size for s in specs) == 159_383_552
    return specs


def c2_kernarg(va: dict, layer: int = 0, ctx: int = 4096, ctx_len: int = 3072) -> bytes:
    """kc_fixture_decode_attn(q, k, v, out, scratch, layer, ctx, ctx_len)."""
    return struct.pack("<QQQQQiii", va["q"], va["k_cache"], va["v_cache"], va["attn_out"], va["workspace"], layer,
                       ctx, ctx_len)


# ------------------------------------------------------------------ c3
C3_SHAPE = (8, 16, 16384, 128)          # paper's B2 H16 S4096 D128 scaled in B and S
C3_BUF_BYTES = 8 * 16 * 16384 * 128 * 2  # 536,870,912 B per tensor
C3_MISMATCH_P = 0.113                    # the paper's 11.3%
C3_K_FLIP_OFFSET = 65536 * 1000 + 17


# ------------------------------------------------------------------ c4
C4_TOTAL = 30_074_000_000                # PAPER.md:1285 (vLLM, 30,074 MB)
C4_LAYERS = 24
C4_EXPERTS = 60
C4_W13 = (60, 2816, 2048)                # Qwen1.5-MoE-A2.7B gate/up (reading R24)
C4_W2 = (60, 2048, 1408)
C4_W13_BYTES = 60 * 2816 * 2048 * 2      # 692,060,160
C4_W2_BYTES = 60 * 2048 * 1408 * 2       # 346,030,080
C4_PTR_BYTES = 4096
C4_T = 16                                # tokens of the F3 dispatch
C4_N_MISC = 113


def c4_specs() -> list:
    """185 regions: 24 x (w13, w2, ptr_table) + 113 misc, sum exactly 30,074,000,000 B."""
    rng = np.random.default_rng(seed(4))
    specs = []
    for layer in range(C4_LAYERS):
        specs.append(RegionSpec(f"w13_{layer}", C4_W13_BYTES, "bf16", "normal", {"std": 0.02}, layer))
        specs.append(RegionSpec(f"w2_{layer}", C4_W2_BYTES, "bf16", "normal", {"std": 0.02}, layer))
        specs.append(RegionSpec(f"ptr_{layer}", C4_PTR_BYTES, "u64", "ptr_table", {}, layer))
    misc_total = C4_TOTAL - len(specs) // 3 * (C4_W13_BYTES + C4_W2_BYTES + C4_PTR_BYTES)
    fixed = [RegionSpec("x", 65536, "bf16", "normal", {"std": 1.0}),
             RegionSpec("topk", 65536, "i32", "topk", {}),
             RegionSpec("y", C4_T * 2816 * 4, "f32", "zero")]
    rest = misc_total - sum(s.size for s in fixed)
    n = C4_N_MISC - len(fixed)
    lo, hi = math.log(64 * 1024), math.log(256 * 2**20)
    raw = np.exp(rng.uniform(lo, hi, size=n))
    sizes = np.floor(raw / raw.sum() * rest / 2).astype(np.int64) * 2     # even (bf16 elements)
    sizes[-1] += rest - int(sizes.sum())
    zero = rng.random(n) < 0.10                                            # 10% of misc zero-filled
    misc = [RegionSpec(f"misc_{i}", int(sz), "bf16", "zero" if z else "normal", {"std": 1.0})
            for i, (sz, z) in enumerate(zip(sizes, zero))]
    specs += fixed + misc
    assert len(specs) == 185 and sum(s.size for s in specs) == C4_TOTAL
    return specs


def c4_placement(specs: list, n_gpus: int) -> list:
    """E1 residency-first placement: layer l on GPU l mod N, misc to the least loaded."""
    load = [0] * n_gpus
    owner = []
    for s in specs:
        g = s.layer % n_gpus if s.layer >= 0 else None
        owner.append(g)
        if g is not None:
            load[g] += s.size
    for i, s in enumerate(specs):
        if owner[i] is None:
            g = min(range(n_gpus), key=lambda j: load[j])
            owner[i] = g
            load[g] += s.size
    return owner


def c4_topk(s: int | None = None) -> np.ndarray:
    """Seeded top-2 routing of T tokens over 60 experts."""
    rng = np.random.default_rng(seed(4, 7) if s is None else s)
    out = np.zeros((C4_T, 2), dtype=np.int32)
    for t in range(C4_T):
        out[t] = rng.choice(C4_EXPERTS, size=2, replace=False)
    return out


def c4_ptr_table(w13_va: int, w2_va: int) -> np.ndarray:
    """60 w13 expert pointers then 60 w2 expert pointers (device VAs), zero padded to 4 KiB."""
    t = np.zeros(C4_PTR_BYTES // 8, dtype=np.uint64)
    t[:60] = np.uint64(w13_va) + np.uint64(2816 * 2048 * 2) * np.arange(60, dtype=np.uint64)
    t[60:120] = np.uint64(w2_va) + np.uint64(2048 * 1408 * 2) * np.arange(60, dtype=np.uint64)
    return t


def c4_kernarg(ptr_va: int, x_va: int, topk_va: int, y_va: int) -> bytes:
    """kc_fixture_moe_gemv(ptr_table, x, topk, y, T, O, I)."""
    return struct.pack("<QQQQiii", ptr_va, x_va, topk_va, y_va, C4_T, 2816, 2048)


# ------------------------------------------------------------------ c5
C5_SIZES = [4096, 65536, 2**20, 16 * 2**20, 256 * 2**20, 4 * 2**30]
C5_COUNTS = [10, 100, 1000, 10000, 100000]
C5_CAP = 48 * 2**30


def c5_cells() -> list:
    return [(S, n) for S in C5_SIZES for n in C5_COUNTS if S * n <= C5_CAP]


def c5_sizes(S: int, n: int, jitter: bool, s: int | None = None) -> np.ndarray:
    rng = np.random.default_rng(seed(5) if s is None else s)
    base = np.full(n, S, dtype=np.int64)
    if jitter:
        base += rng.integers(0, 4096, size=n)
    return base


# ------------------------------------------------------------------ F4 (drift study)
# The attn_fwd shape the paper measures: fp16, B=2, H=16,
# S=4096, D=128.  Inputs N(0, 0.5) as in the Triton attention tutorial's test
# (reading R32); sm_scale = 1/sqrt(D).  Seed 260503208 + 6 (stream 0/1/2 = Q/K/V).
F4_B, F4_H, F4_S, F4_D = 2, 16, 4096, 128
F4_STD = 0.5
F4_SM_SCALE = 1.0 / math.sqrt(F4_D)
F4_BLOCK_M = 64
F4_BYTES = F4_B * F4_H * F4_S * F4_D * 2          # 33,554,432 B per tensor
F4_SPECS = [RegionSpec(n, F4_BYTES, dtype="f16", fill=("zero" if n == "o" else "normal"), params={"std": F4_STD})
            for n in ("q", "k", "v", "o")]


def f4_cubin(block_n: int) -> str:
    """Code object of the attn_fwd fixture compiled for one BLOCK_N "autotune config"."""
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), f"kc_attn_fwd_n{block_n}.cubin")


def f4_launch(B: int = F4_B, H: int = F4_H, S: int = F4_S) -> dict:
    """Grid/block of kc_fixture_attn_fwd: one CTA of 256 threads per 64 query rows and head."""
    return {"grid": (S // F4_BLOCK_M, B * H, 1), "block": (256, 1, 1)}


def f4_kernarg(q_va: int, k_va: int, v_va: int, o_va: int, S: int = F4_S, sm_scale: float = F4_SM_SCALE) -> bytes:
    """kc_fixture_attn_fwd(Q, K, V, O, int S, float sm_scale): natural alignment 8,8,8,8,4,4."""
    return struct.pack("<QQQQif", q_va, k_va, v_va, o_va, S, sm_scale)


# ------------------------------------------------------------------ torch materialisation
class _CAI:
    """Expose a raw device range through __cuda_array_interface__ (zero-copy torch view)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def dev_view(ptr: int, nbytes: int, device: int = 0):
    """uint8 torch tensor aliasing [ptr, ptr+nbytes) on cuda:device (plumbing only)."""
    import torch
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(ptr, nbytes), device=f"cuda:{device}")


def fill_device(view, spec: RegionSpec, gen) -> None:
    """Fill a uint8 device view with the spec's recipe using torch's device Philox generator."""
    import torch
    n = view.numel()
    if spec.fill == "zero" or n == 0:
        view.zero_()
        return
    if spec.fill == "u8":
        view.copy_(torch.randint(0, 256, (n,), dtype=torch.uint8, device=view.device, generator=gen))
        return
    if spec.fill == "u8range":
        lo, hi = spec.params["lo"], spec.params["hi"]
        view.copy_(torch.randint(lo, hi + 1, (n,), dtype=torch.uint8, device=view.device, generator=gen))
        return
    if spec.fill == "arange_i32":
        view.view(torch.int32).copy_(torch.arange(n // 4, dtype=torch.int32, device=view.device))
        return
    if spec.fill == "normal":
        std = spec.params.get("std", 1.0)
        tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[spec.dtype]
        es = torch.tensor([], dtype=tdt).element_size()
        m = n // es
        step = 1 << 27
        out = view[: m * es].view(tdt)
        for o in range(0, m, step):
            k = min(step, m - o)
            out[o:o + k].copy_((torch.randn(k, device=view.device, generator=gen) * std).to(tdt))
        if n > m * es:
            view[m * es:].zero_()
        return
    if spec.fill == "kv":
        valid, ctx = spec.params["valid"], spec.params["ctx"]
        t = view.view(torch.float16).view(-1, ctx, 64)          # [L*KVH][ctx][64]
        t.copy_(torch.randn(t.shape, device=view.device, generator=gen).to(torch.float16))
        t[:, valid:, :] = 0
        return
    raise ValueError(f"fill recipe {spec.fill!r} needs explicit contents")


F16_BITS = {"maxfin": 0x7BFF, "inf": 0x7C00, "qnan": 0x7E00}
BF16_BITS = {"maxfin": 0x7F7F, "inf": 0x7F80, "qnan": 0x7FC0}


def special_positions(n: int) -> list:
    """Fixed element indices of the c3 specials (spread over the buffer)."""
    step = max(1, n // 9)
    return [min(n - 1, step * j + 17) for j in range(1, 9)]


def plant_c3(ref16, act16, kind: str, p: float, gen, specials: bool = True) -> None:
    """c3 planting recipe on int16 torch views of 16-bit floats.

    act = ref, then Bernoulli(p) elements get their magnitude bits shifted by
    +-k (k = 1 w.p. 0.9, else U{2..16}), clamped to stay finite.  Specials at
    fixed indices: 3 x A = NaN where R is finite; both NaN with the same payload;
    both NaN with different payloads; A = +inf; R = +0 / A = -0; R = 0 / A = min
    subnormal; A = -R at argmax |R|."""
    import torch
    B = F16_BITS if kind == "f16" else BF16_BITS
    n = ref16.numel()
    dev = ref16.device
    m = torch.rand(n, device=dev, generator=gen) < p
    k = torch.where(torch.rand(n, device=dev, generator=gen) < 0.9, torch.ones(n, dtype=torch.int32, device=dev),
                    torch.randint(2, 17, (n,), dtype=torch.int32, device=dev, generator=gen))
    sgn = torch.where(torch.rand(n, device=dev, generator=gen) < 0.5, -1, 1).to(torch.int32)
    bits = ref16.to(torch.int32) & 0xFFFF
    newbits = (bits & 0x8000) | torch.clamp((bits & 0x7FFF) + sgn * k, min=0, max=B["maxfin"])
    newbits = torch.where(newbits >= 0x8000, newbits - 0x10000, newbits).to(torch.int16)
    act16.copy_(torch.where(m, newbits, ref16))
    del m, k, sgn, bits, newbits
    if not specials or n < 64:
        return

    def i16(v):
        return v - 0x10000 if v >= 0x8000 else v

    pos = special_positions(n)
    for j in range(3):                         # A = NaN, R finite
        act16[pos[j]] = i16(B["qnan"] | (j + 1))
    ref16[pos[3]] = i16(B["qnan"]); act16[pos[3]] = i16(B["qnan"])          # both NaN, same payload
    ref16[pos[4]] = i16(B["qnan"] | 1); act16[pos[4]] = i16(B["qnan"] | 2)  # both NaN, different payloads
    act16[pos[5]] = i16(B["inf"])              # A = +inf
    ref16[pos[6]] = 0; act16[pos[6]] = i16(0x8000)                           # +0 vs -0
    ref16[pos[7]] = 0; act16[pos[7]] = 1                                     # 0 vs min subnormal
    fl = ref16.view(torch.float16 if kind == "f16" else torch.bfloat16).float().abs()
    fl = torch.nan_to_num(fl, nan=0.0)
    am = int(torch.argmax(fl))
    act16[am] = i16((int(ref16[am]) & 0xFFFF) ^ 0x8000)                      # A = -R at argmax |R|
