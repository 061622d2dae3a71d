// kc_kernels.cu -- the data-parallel hot path of Kerncap's capture-and-validate
// loop on B200 (sm_100a): K1 chunked XXH64 content hash (cp.async-staged rings,
// 4 lanes per chunk, shuffle merge; TMA bulk rings as measured alternatives),
// K6 = K1 + copy into a snapshot arena, region/snapshot digests, K3 written
// set, K2 fused diff (bitmap, counts, ULP, fp64 abs/rel, allclose, NaN
// counters), K5 fused hash + compare, K4 gather.
//
// Definitions: SURVEY.md 8(c) O2-O4 and DESIGN.md readings R1-R34, restating
// PAPER.md:681-691 (chunked snapshot), 1120-1126 (byte-exact compare),
// 1128-1135 (allclose + explicit NaN reporting).  Compiled WITHOUT fast-math
// and with -fmad=false; every fp64 op below is an explicit _rn intrinsic.
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kc_kernels.cuh"

// KC_CHECKS=1 (libkc_checked.so, `python -m paper_2605_03208_b200.build --checked`): device-side
// bounds checks on every shared-memory ring slot, queue push and chunk lookup of the hot path,
// trapping with the failing condition.  The GPU pool has compute-sanitizer disabled, so the
// checked build run under the parity tests stands in for memcheck on these kernels.
#ifndef KC_CHECKS
#define KC_CHECKS 0
#endif
#if KC_CHECKS
#include <cstdio>
#define KC_DCHECK(c)                                                                                    \
    do {                                                                                                \
        if (!(c)) {                                                                                     \
            printf("KC_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #c, __FILE__, __LINE__,       \
                   (int)blockIdx.x, (int)threadIdx.x);                                                  \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#else
#define KC_DCHECK(c) ((void)0)
#endif

namespace kc {

// ========================================================================== //
// XXH64 primitives (public algorithm; constants SURVEY.md Appendix A)         //
// ========================================================================== //
#define P1 0x9E3779B185EBCA87ULL
#define P2 0xC2B2AE3D27D4EB4FULL
#define P3 0x165667B19E3779F9ULL
#define P4 0x85EBCA77C2B2AE63ULL
#define P5 0x27D4EB2F165667C5ULL

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// accumulator round: rotl(acc + x*P2, 31) * P1
__device__ __forceinline__ uint64_t xround(uint64_t acc, uint64_t x) {
    acc += x * P2;
    acc = rotl64(acc, 31);
    return acc * P1;
}

// The accumulator chain in "y form".  With y = acc + x*P2 (the pre-rotation
// sum) the round is  y' = rotl(y, 31)*P1 + x'*P2,  and the 64-bit multiply's
// low product absorbs the next word's x'*P2 as its 64-bit addend (one
// mad.wide.u32).  x'*P2 is off the chain (tools/probes/k1_round_probe.cu:
// ~30 cycles per round for one chain per thread at one warp per SMSP, every
// formulation within 15%; this one is the fastest measured).
// A lane starts from y0 = rotr(seed * P1^-1, 31), so that rotl(y0, 31)*P1 is
// the XXH64 lane seed, and ends with yfinal(y) = rotl(y, 31)*P1 = the lane's
// accumulator.  Same arithmetic mod 2^64, reordered: results are identical.
__device__ __forceinline__ uint64_t ystep(uint64_t y, uint64_t x) {
    // one PTX block: x*P2 is formed completely off the chain (plo, phi), and the
    // chain is  funnel shifts -> mad (rh*P1lo + phi) -> mad (rl*P1hi + .) ->
    // mad.lo.cc / madc.hi (rl*P1lo + {plo, .}): four dependent SASS per stripe
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh, yl, yh, plo, phi, rl, rh, t;\n\t"
        "mov.b64 {xl, xh}, %2;\n\t"
        "mov.b64 {yl, yh}, %3;\n\t"
        "mul.lo.u32 plo, xl, %4;\n\t"
        "mul.hi.u32 phi, xl, %4;\n\t"
        "mad.lo.u32 phi, xl, %5, phi;\n\t"
        "mad.lo.u32 phi, xh, %4, phi;\n\t"
        "shf.l.wrap.b32 rh, yl, yh, 31;\n\t"
        "shf.l.wrap.b32 rl, yh, yl, 31;\n\t"
        "mad.lo.u32 t, rh, %6, phi;\n\t"
        "mad.lo.u32 t, rl, %7, t;\n\t"
        "mad.lo.cc.u32 %0, rl, %6, plo;\n\t"
        "madc.hi.u32 %1, rl, %6, t;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "l"(y), "r"((uint32_t)P2), "r"((uint32_t)(P2 >> 32)), "r"((uint32_t)P1),
          "r"((uint32_t)(P1 >> 32)));
    return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t yfinal(uint64_t y) { return ystep(y, 0); }

__device__ __forceinline__ uint64_t xavalanche(uint64_t h) {
    h ^= h >> 33;
    h *= P2;
    h ^= h >> 29;
    h *= P3;
    h ^= h >> 32;
    return h;
}

// unaligned little-endian loads from global memory (byte-assembled)
__device__ __forceinline__ uint64_t ldg_u64_bytes(const uint8_t* p) {
    uint64_t v = 0;
#pragma unroll
    for (int i = 7; i >= 0; --i) v = (v << 8) | __ldg(p + i);
    return v;
}
__device__ __forceinline__ uint32_t ldg_u32_bytes(const uint8_t* p) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 3; i >= 0; --i) v = (v << 8) | __ldg(p + i);
    return v;
}

// Finish XXH64 on a quad: v = this lane's accumulator (lane ql of 4), len the
// total length, tail = pointer to the bytes after the last full stripe.
// All 4 lanes must call; every lane returns the same hash.
template <bool ALIGNED>
__device__ __forceinline__ uint64_t quad_finish(uint64_t v, int ql, unsigned qmask, uint64_t len, const uint8_t* tail) {
    uint64_t h;
    if (len >= 32) {
        const int rot = ql == 0 ? 1 : (ql == 1 ? 7 : (ql == 2 ? 12 : 18));
        uint64_t a = rotl64(v, rot);
        a += __shfl_xor_sync(qmask, a, 1, 4);
        a += __shfl_xor_sync(qmask, a, 2, 4);
        const uint64_t m = xround(0, v);
        const uint64_t m0 = __shfl_sync(qmask, m, 0, 4);
        const uint64_t m1 = __shfl_sync(qmask, m, 1, 4);
        const uint64_t m2 = __shfl_sync(qmask, m, 2, 4);
        const uint64_t m3 = __shfl_sync(qmask, m, 3, 4);
        h = a;
        h = (h ^ m0) * P1 + P4;
        h = (h ^ m1) * P1 + P4;
        h = (h ^ m2) * P1 + P4;
        h = (h ^ m3) * P1 + P4;
    } else {
        h = P5;  // seed 0
    }
    h += len;
    uint32_t rem = (uint32_t)(len & 31);
    const uint8_t* p = tail;
    while (rem >= 8) {
        const uint64_t x = ALIGNED ? __ldg(reinterpret_cast<const unsigned long long*>(p)) : ldg_u64_bytes(p);
        h ^= xround(0, x);
        h = rotl64(h, 27) * P1 + P4;
        p += 8;
        rem -= 8;
    }
    if (rem >= 4) {
        const uint32_t x = ALIGNED ? __ldg(reinterpret_cast<const unsigned int*>(p)) : ldg_u32_bytes(p);
        h ^= (uint64_t)x * P1;
        h = rotl64(h, 23) * P2 + P3;
        p += 4;
        rem -= 4;
    }
    while (rem > 0) {
        h ^= (uint64_t)__ldg(p) * P5;
        h = rotl64(h, 11) * P1;
        ++p;
        --rem;
    }
    return xavalanche(h);
}

__device__ __forceinline__ uint64_t lane_yseed(int ql) {
    // y0 = rotr(v * P1^-1, 31) for the seed-0 lane seeds v1 = P1+P2, v2 = P2,
    // v3 = 0, v4 = -P1 (P1^-1 = 0x0887493432BADB37 mod 2^64)
    return ql == 0 ? 0x32E245F52D5533D6ULL : (ql == 1 ? 0x32E245F32D5533D6ULL : (ql == 2 ? 0ULL : ~0ULL));
}

// XXH64 of one contiguous global byte range by a quad, direct loads (16
// stripes of loads in flight per lane on the aligned path: the digests walk
// manifests of up to ~84 KB serially, so load latency must not be exposed).
template <bool ALIGNED>
__device__ uint64_t quad_xxh64_global(const uint8_t* p, uint64_t len, int ql, unsigned qmask) {
    uint64_t v = lane_yseed(ql);  // y form
    const uint64_t nst = len >= 32 ? len / 32 : 0;
    const uint8_t* q = p + 8 * ql;
    uint64_t t = 0;
    if (ALIGNED) {
        // software-pipelined: batch k+1's 16 loads are in flight while batch k is hashed
        constexpr int U = 16;
        const unsigned long long* g = reinterpret_cast<const unsigned long long*>(q);
        if (nst >= 2 * U) {
            uint64_t xa[U], xb[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xa[u] = __ldg(g + 4 * u);
            for (; t + 2 * U <= nst; t += 2 * U) {
#pragma unroll
                for (int u = 0; u < U; ++u) xb[u] = __ldg(g + 4 * (t + U + u));
#pragma unroll
                for (int u = 0; u < U; ++u) v = ystep(v, xa[u]);
                if (t + 3 * U <= nst) {
#pragma unroll
                    for (int u = 0; u < U; ++u) xa[u] = __ldg(g + 4 * (t + 2 * U + u));
                }
#pragma unroll
                for (int u = 0; u < U; ++u) v = ystep(v, xb[u]);
            }
            if (t + U <= nst) {  // xa already holds batch t when fewer than 2U stripes remain
#pragma unroll
                for (int u = 0; u < U; ++u) v = ystep(v, xa[u]);
                t += U;
            }
        }
    }
    for (; t < nst; ++t) {
        const uint64_t x =
            ALIGNED ? __ldg(reinterpret_cast<const unsigned long long*>(q + 32 * t)) : ldg_u64_bytes(q + 32 * t);
        v = ystep(v, x);
    }
    return quad_finish<ALIGNED>(yfinal(v), ql, qmask, len, p + 32 * nst);
}

__device__ __forceinline__ int find_region(const RegionDev* __restrict__ r, int n, uint64_t g) {
    int lo = 0, hi = n;  // first i with chunk_off > g, minus one
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (r[mid].chunk_off <= g) lo = mid + 1; else hi = mid;
    }
    return lo - 1;
}

// ========================================================================== //
// K1: chunk hash.  XXH64 of a 64 KiB chunk is four serial 2,048-step chains //
// (one per accumulator), so K1 is latency-bound per chunk and HBM-bound only //
// with >= ~64 chunks in flight per SM.  A quad of lanes hashes one chunk (one //
// accumulator per lane, shuffle merge).  Two staging designs share the body: //
//  * k1_hash_tma: per-quad 3-stage ring filled by cp.async.bulk (TMA 1-D     //
//    bulk copies + mbarrier complete_tx), lane 0 of the quad the producer;   //
//  * k1_hash_cpasync (default): a warp stages its 8 quads' next slices with  //
//    coalesced 16-byte cp.async (512 B per warp instruction) into padded,    //
//    bank-conflict-free rings.                                               //
// Measured on B200: the per-request cost of 1 KiB bulk copies    //
// caps the TMA ring at ~5.0 TB/s, the cp.async ring reaches the HBM peak.    //
// ========================================================================== //
template <int THREADS, int STAGES, int SLICE>
struct HkCfg {
    static constexpr int kThreads = THREADS;
    static constexpr int kSlots = THREADS / 4;
    static constexpr int kStages = STAGES;
    static constexpr int kSlice = SLICE;
    static constexpr int kPitch = SLICE + 32;  // quads of a warp land on distinct bank groups
    static constexpr size_t kSmem = (size_t)kSlots * STAGES * kPitch + (size_t)kSlots * STAGES * 8;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

struct ChunkRef {
    const uint8_t* src;
    uint32_t len;
};

// chunk -> region: one load from the host-built map when given (uploaded once
// with the cached region table), else binary search over the chunk offsets
__device__ __forceinline__ ChunkRef chunk_ref(const RegionDev* __restrict__ regs, int nreg, uint64_t g,
                                             const uint32_t* __restrict__ map) {
    const int r = map ? (int)__ldg(map + g) : find_region(regs, nreg, g);
    KC_DCHECK(r >= 0 && r < nreg && regs[r].chunk_off <= g);
    const uint64_t off = (g - regs[r].chunk_off) * kChunk;
    KC_DCHECK(off < regs[r].size);
    const uint64_t rem = regs[r].size - off;
    return {reinterpret_cast<const uint8_t*>(regs[r].base + off), rem < kChunk ? (uint32_t)rem : (uint32_t)kChunk};
}

template <class CFG>
__global__ void __launch_bounds__(CFG::kThreads, 1)
    k1_hash_tma(const RegionDev* __restrict__ regs, int nreg, uint64_t C, uint64_t* __restrict__ out,
                const uint32_t* __restrict__ map) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int slot = threadIdx.x >> 2;
    const int ql = threadIdx.x & 3;
    const unsigned qmask = 0xFu << (threadIdx.x & 28);
    uint8_t* ring = smem + (size_t)slot * CFG::kStages * CFG::kPitch;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)CFG::kSlots * CFG::kStages * CFG::kPitch) + slot * CFG::kStages;

    if (ql == 0) {
#pragma unroll
        for (int s = 0; s < CFG::kStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

    const uint64_t Q = (uint64_t)CFG::kSlots * gridDim.x;
    const uint64_t g0 = (uint64_t)slot * gridDim.x + blockIdx.x;

    // ---- producer cursor (used by ql == 0 only) ----
    uint64_t pg = g0;              // chunk being fetched
    const uint8_t* psrc = nullptr; // its first byte
    uint32_t pbytes = 0, poff = 0; // stripe bytes to stage, bytes already issued
    bool phave = false;
    uint32_t fetched = 0;
    auto issue_next = [&]() {
        while (pg < C) {
            if (!phave) {
                const ChunkRef cr = chunk_ref(regs, nreg, pg, map);
                psrc = cr.src;
                pbytes = cr.len >= 32 ? (cr.len & ~31u) : 0u;
                poff = 0;
                phave = true;
            }
            if (poff < pbytes) {
                const uint32_t b = min((uint32_t)CFG::kSlice, pbytes - poff);
                const int st = fetched % CFG::kStages;
                mbar_arrive_expect_tx(&bars[st], b);
                bulk_g2s(ring + st * CFG::kPitch, psrc + poff, b, &bars[st], policy);
                poff += b;
                ++fetched;
                if (poff == pbytes) { pg += Q; phave = false; }
                return;
            }
            pg += Q;
            phave = false;
        }
    };
    if (ql == 0) {
        for (int s = 0; s < CFG::kStages; ++s) issue_next();
    }

    uint32_t consumed = 0;
    for (uint64_t g = g0; g < C; g += Q) {
        const ChunkRef cr = chunk_ref(regs, nreg, g, map);
        const uint32_t nst = cr.len >= 32 ? cr.len / 32 : 0;
        uint64_t v = lane_yseed(ql);  // y form
        uint32_t remaining = nst * 32;
        while (remaining > 0) {
            const int st = consumed % CFG::kStages;
            mbar_wait(&bars[st], (consumed / CFG::kStages) & 1);
            const uint64_t* p = reinterpret_cast<const uint64_t*>(ring + st * CFG::kPitch) + ql;
            if (remaining >= (uint32_t)CFG::kSlice) {
#pragma unroll
                for (int t = 0; t < CFG::kSlice / 32; ++t) v = ystep(v, p[4 * t]);
                remaining -= CFG::kSlice;
            } else {
                const uint32_t n = remaining / 32;
                for (uint32_t t = 0; t < n; ++t) v = ystep(v, p[4 * t]);
                remaining = 0;
            }
            ++consumed;
            __syncwarp(qmask);  // all 4 lanes are done with this stage
            if (ql == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_next();
            }
        }
        const uint64_t h = quad_finish<true>(yfinal(v), ql, qmask, cr.len, cr.src + (size_t)nst * 32);
        if (ql == 0) out[g] = h;
    }
}

// V_CPASYNC: warp-cooperative cp.async staging.  A warp hashes 8 consecutive
// chunks (one per quad); per pipeline step every lane copies 16-byte pieces of
// all 8 chunks' next 1 KiB slices (coalesced 512-byte rows), so 64 chunks per
// SM are in compute while STAGES-1 steps are in flight.  Slices are padded by
// 32 bytes so the 8 quads of a warp read distinct bank groups.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// the same with a shared-window address computed once per thread: cvta per
// copy cost S2R SR_CgaCtaId + MOV + LEA under each copy's predicate (K1's
// staging was 8 SASS per 16-byte copy, 17% of the sub-wave K1's samples)
// KC_CP_L2_PREFETCH=1 adds the .L2::256B prefetch qualifier: measured neutral
// on B200 (K1 over 2 GiB 6,394 vs 6,357 GB/s; the 30 GB pool 6,633 vs 6,623;
// K5 6,264 vs 6,282), so off by default
#ifndef KC_CP_L2_PREFETCH
#define KC_CP_L2_PREFETCH 0
#endif
__device__ __forceinline__ void cp_async16_s(uint32_t saddr, const void* gmem) {
#if KC_CP_L2_PREFETCH
    // L2::256B: the L2 fetches whole 256-byte blocks (a warp's copy instruction
    // covers 512 contiguous bytes of one chunk)
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(saddr), "l"(gmem) : "memory");
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Slice layout in the ring.  SWZ = 0 (round 2): quad q's slice at q * (SL + 32), so the 8 quads
// of a warp read distinct bank groups; but then a 128-byte global line lands across two
// 128-byte shared rows for 3 quads in 4, and L1TEX splits its cp.async into two L2 requests
// that touch 3 sectors each (ncu: 7 requests and 22 sectors per 512-byte LDGSTS instead of 4
// and 16; 1.375 x the L2 sector traffic, 20% L2 hits).  SWZ = 1: slices at q * SL, 128-byte
// aligned, and within every 128-byte row stripe t of quad q sits at position (t ^ q) & 3
// (byte offset ^ (q & 3) << 5): each global line fills exactly one shared row, and the quads'
// words of one round spread over 4 bank groups (quads q and q + 4 share one: 2 wavefronts for
// the warp's 256 bytes, the minimum).
__host__ __device__ constexpr int swz_off(bool swz, int q, int off) { return swz ? off ^ ((q & 3) << 5) : off; }

template <int WARPS, int STAGES, int SL, bool SWZ = true>
struct CpCfg {
    static constexpr int kWarps = WARPS, kStages = STAGES, kSlice = SL;
    static constexpr bool kSwz = SWZ;
    static constexpr int kPitch = SWZ ? SL : SL + 32;  // see swz_off
    static constexpr int kWStage = 8 * kPitch;  // one warp's stage: 8 chunk slices
    static constexpr int kUPC = SL / 16;        // 16-byte copy units per chunk slice
    static constexpr int kUPL = (8 * kUPC + 31) / 32;  // copy units per lane per step
    static constexpr size_t kSmem = (size_t)WARPS * STAGES * kWStage;
};

// COPY (K6, the fused capture pass): the staged slices are also written to the
// snapshot arena (dst[r] = arena address of region r's byte 0) with streaming
// 16-byte stores, so one HBM read of every region yields both its manifest and
// its stored copy.  Each 1 KiB slice is written by two warp-wide 512 B rows.
__device__ __forceinline__ void st_cs16(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

template <class CFG, bool COPY = false>
__global__ void __launch_bounds__(CFG::kWarps * 32, 1)
    k1_hash_cpasync(const RegionDev* __restrict__ regs, int nreg, uint64_t C, uint64_t* __restrict__ out,
                    const uint32_t* __restrict__ map, const unsigned long long* __restrict__ dst = nullptr,
                    const uint32_t* __restrict__ order = nullptr) {
    static_assert(!COPY || CFG::kUPC % 32 == 0, "K6 copy-out maps copy unit k to chunk 32k / UPC");
    constexpr int WARPS = CFG::kWarps, STAGES = CFG::kStages, SL = CFG::kSlice, PITCH = CFG::kPitch;
    constexpr int WSTAGE = CFG::kWStage, UPC = CFG::kUPC, UPL = CFG::kUPL;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, q = lane >> 2, ql = lane & 3;
    const unsigned qmask = 0xFu << (lane & 28);
    uint8_t* wring = smem + (size_t)w * STAGES * WSTAGE;
    const uint32_t wring_s = smem_u32(wring);
    const uint64_t ngroups = (C + 7) / 8;
    const uint64_t W = (uint64_t)gridDim.x * WARPS;
    const uint64_t j0 = (uint64_t)w * gridDim.x + blockIdx.x;  // interleaved over CTAs

    // fetch cursor (warp-uniform): group jf, slice sf.  Per lane: the chunk of
    // each of its UPL copy units (unit u = lane + 32k -> chunk u / UPC).
    uint64_t jf = j0;
    uint32_t sf = 0, f_nsl = 0;
    unsigned long long u_src[UPL];
    uint32_t u_bytes[UPL];
    // position i of the chunk sequence -> chunk index (length-sorted order, or identity)
    auto chunk_at = [&](uint64_t i) -> uint64_t { return order && i < C ? (uint64_t)__ldg(order + i) : i; };
    auto load_group = [&](uint64_t j) {
        const uint64_t g = chunk_at(8 * j + q);
        unsigned long long src = 0;
        uint32_t bytes = 0;
        if (g < C) {
            const ChunkRef cr = chunk_ref(regs, nreg, g, map);
            src = (unsigned long long)cr.src;
            bytes = cr.len >= 32 ? (cr.len & ~31u) : 0u;
        }
        f_nsl = __reduce_max_sync(0xFFFFFFFFu, (bytes + SL - 1) / SL);
#pragma unroll
        for (int k = 0; k < UPL; ++k) {
            const int u = lane + 32 * k;
            const int qq = u < 8 * UPC ? u / UPC : 0;
            u_src[k] = __shfl_sync(0xFFFFFFFFu, src, 4 * qq);
            u_bytes[k] = __shfl_sync(0xFFFFFFFFu, bytes, 4 * qq);
        }
    };
    auto issue = [&](int stage) {
        const uint32_t dst = wring_s + stage * WSTAGE;
#pragma unroll
        for (int k = 0; k < UPL; ++k) {
            const int u = lane + 32 * k;
            if (u < 8 * UPC) {
                const int qq = u / UPC, off = (u % UPC) * 16;  // qq is k * 32 / UPC: compile-time
                const uint32_t g_off = sf * SL + off;
                if (g_off < u_bytes[k]) {
                    KC_DCHECK(dst + qq * PITCH + swz_off(CFG::kSwz, qq, off) + 16 <= wring_s - w * STAGES * WSTAGE +
                                                                                       CFG::kSmem);
                    KC_DCHECK(g_off + 16 <= u_bytes[k]);
                    cp_async16_s(dst + qq * PITCH + swz_off(CFG::kSwz, qq, off),
                                 reinterpret_cast<const uint8_t*>(u_src[k]) + g_off);
                }
            }
        }
    };
    auto advance = [&]() {
        if (++sf >= f_nsl) {
            sf = 0;
            jf += W;
            if (jf < ngroups) load_group(jf); else f_nsl = 0;
        }
    };
    auto fetch = [&](int stage) {  // next step of the sequence (skips groups with no full stripe)
        while (jf < ngroups && f_nsl == 0) {
            jf += W;
            if (jf < ngroups) load_group(jf);
        }
        if (jf < ngroups) {
            issue(stage);
            advance();
        }
        cp_async_commit();
    };
    if (j0 < ngroups) load_group(jf);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) fetch(s);
    uint32_t step = 0;
    for (uint64_t j = j0; j < ngroups; j += W) {
        const uint64_t g = chunk_at(8 * j + q);
        ChunkRef cr = {nullptr, 0};
        if (g < C) cr = chunk_ref(regs, nreg, g, map);
        const uint32_t nst = cr.len >= 32 ? cr.len / 32 : 0;
        const uint32_t nsl = __reduce_max_sync(0xFFFFFFFFu, (nst * 32 + SL - 1) / SL);
        // K6: arena address of this quad's chunk (0 past the end)
        unsigned long long cdst = 0;
        if (COPY && g < C) {
            const int r = map ? (int)__ldg(map + g) : find_region(regs, nreg, g);
            cdst = dst[r] + (g - regs[r].chunk_off) * kChunk;
        }
        uint64_t v = lane_yseed(ql);  // y form
        for (uint32_t s = 0; s < nsl; ++s, ++step) {
            cp_async_wait<STAGES - 2>();
            __syncwarp();
            const int st = step % STAGES;
            const uint64_t* p = reinterpret_cast<const uint64_t*>(wring + st * WSTAGE + q * PITCH) + ql;
            const uint32_t done = s * (SL / 32);
            const uint32_t n = nst > done ? min((uint32_t)(SL / 32), nst - done) : 0u;
            const int sq = CFG::kSwz ? (q & 3) : 0;  // stripe t of this quad at row position t ^ sq
            KC_DCHECK(reinterpret_cast<const uint8_t*>(p) - smem + 32 * (SL / 32 - 1) + 8 <= (long)CFG::kSmem);
            if (n == SL / 32) {
                const uint64_t* pb[4] = {p + 4 * (0 ^ sq), p + 4 * (1 ^ sq), p + 4 * (2 ^ sq), p + 4 * (3 ^ sq)};
#pragma unroll
                for (int t = 0; t < SL / 32; ++t) v = ystep(v, pb[t & 3][4 * (t & ~3)]);
            } else {
                for (uint32_t t = 0; t < n; ++t) v = ystep(v, p[4 * (t ^ sq)]);
            }
            if (COPY) {  // the stage's 8 slices -> the arena, before the slot is refilled
#pragma unroll
                for (int k = 0; k < UPL; ++k) {
                    const int qq = (32 * k) / UPC;
                    const int off = ((32 * k) % UPC + lane) * 16;
                    const unsigned long long d = __shfl_sync(0xFFFFFFFFu, cdst, 4 * qq);
                    const uint32_t b = __shfl_sync(0xFFFFFFFFu, nst * 32, 4 * qq);
                    const uint32_t g_off = s * SL + off;
                    if (g_off < b)
                        st_cs16(reinterpret_cast<uint8_t*>(d) + g_off,
                                *reinterpret_cast<const uint4*>(wring + st * WSTAGE + qq * PITCH +
                                                                swz_off(CFG::kSwz, qq, off)));
                }
            }
            __syncwarp();
            fetch((step + STAGES - 1) % STAGES);
        }
        if (g < C) {
            const uint64_t h = quad_finish<true>(yfinal(v), ql, qmask, cr.len, cr.src + (size_t)nst * 32);
            if (ql == 0) out[g] = h;
            if (COPY && ql == 0)  // the sub-32-byte tail is hashed from global, copy it the same way
                for (uint32_t b = nst * 32; b < cr.len; ++b)
                    reinterpret_cast<uint8_t*>(cdst)[b] = cr.src[b];
        } else {
            quad_finish<true>(yfinal(v), ql, qmask, 0, nullptr);
        }
    }
    cp_async_wait<0>();
}

// ========================================================================== //
// K1, warp-specialized ring (sub-wave snapshots).  Below one wave a chunk's  //
// 2,048-round chain sets the time.  In k1_hash_cpasync the hashing warp also //
// issues its own staging, in order with the chain (~49.5 cycles per round    //
// against ~28-30 for the bare chain, tools/probes/k1_round_probe.cu), and    //
// two chain-bound warps on one SMSP share its FMA pipe (45-50 cycles each).  //
// Here each hashing warp (8 chunks, one per quad) runs alone on its SMSP and //
// a partner producer warp runs the same group/slice sequence, filling the    //
// ring with the same coalesced 16-byte cp.async rows.  A stage is handed     //
// over through two mbarriers: full[st] (32 producer arrivals, each fired by  //
// cp.async.mbarrier.arrive.noinc when that lane's copies have landed) and    //
// empty[st] (one arrival from the hashing warp's lane 0 once the warp is     //
// done reading the slot).  Per 2 KiB slice the hashing warp issues only the  //
// wait, 64 shared loads, 64 rounds and the release.                          //
// ========================================================================== //
// Warp w runs on SMSP w % 4: the hashing warps take slots 0..HW-1 (HW <= 3) and their producers
// slots 3, 7, 11 (all on SMSP 3); the other slots exit at once, so no hashing warp shares its SMSP.
template <int HW, int STAGES, int SL>
struct WsCfg {
    static_assert(HW >= 1 && HW <= 3, "SMSP 3 is left to the producers");
    static constexpr int kHashWarps = HW, kWarps = 4 * HW, kStages = STAGES, kSlice = SL;
    static constexpr bool kSwz = true;
    static constexpr int kPitch = SL;  // swizzled rows (swz_off)
    static constexpr int kWStage = 8 * kPitch;
    static constexpr int kUPC = SL / 16;
    static constexpr int kUPL = (8 * kUPC + 31) / 32;
    static constexpr size_t kRing = (size_t)HW * STAGES * kWStage;
    static constexpr size_t kSmem = kRing + (size_t)HW * STAGES * 2 * sizeof(uint64_t);
};

__device__ __forceinline__ void cp_async_mbar_arrive_noinc_s(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <class CFG>
__global__ void __launch_bounds__(CFG::kWarps * 32, 1)
    k1_hash_ws(const RegionDev* __restrict__ regs, int nreg, uint64_t C, uint64_t* __restrict__ out,
               const uint32_t* __restrict__ map, const uint32_t* __restrict__ order = nullptr) {
    constexpr int HW = CFG::kHashWarps, STAGES = CFG::kStages, SL = CFG::kSlice, PITCH = CFG::kPitch;
    constexpr int WSTAGE = CFG::kWStage, UPC = CFG::kUPC, UPL = CFG::kUPL;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, q = lane >> 2, ql = lane & 3;
    const bool producer = (w & 3) == 3;
    const int hw = producer ? w >> 2 : w;  // the hashing warp this warp is (or serves)
    uint8_t* wring = smem + (size_t)hw * STAGES * WSTAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + CFG::kRing) + hw * 2 * STAGES;
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        uint64_t* b = reinterpret_cast<uint64_t*>(smem + CFG::kRing);
        for (int i = 0; i < HW; ++i)
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&b[i * 2 * STAGES + s], 32);
                mbar_init(&b[i * 2 * STAGES + STAGES + s], 1);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (!producer && w >= HW) return;  // placeholder slot
    const uint64_t ngroups = (C + 7) / 8;
    const uint64_t W = (uint64_t)gridDim.x * HW;
    const uint64_t j0 = (uint64_t)hw * gridDim.x + blockIdx.x;
    auto chunk_at = [&](uint64_t i) -> uint64_t { return order && i < C ? (uint64_t)__ldg(order + i) : i; };

    if (producer) {
        const uint32_t wring_s = smem_u32(wring);
        const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
        // fill k of a stage (k >= 1) waits for the hashing warp's k-th release: parity (k - 1) & 1
        uint32_t st = 0, ph = 0;
        bool first = true;
        for (uint64_t j = j0; j < ngroups; j += W) {
            const uint64_t g = chunk_at(8 * j + q);
            unsigned long long src = 0;
            uint32_t bytes = 0;
            if (g < C) {
                const ChunkRef cr = chunk_ref(regs, nreg, g, map);
                src = (unsigned long long)cr.src;
                bytes = cr.len >= 32 ? (cr.len & ~31u) : 0u;
            }
            const uint32_t nsl = __reduce_max_sync(0xFFFFFFFFu, (bytes + SL - 1) / SL);
            unsigned long long u_src[UPL];
            uint32_t u_bytes[UPL];
#pragma unroll
            for (int k = 0; k < UPL; ++k) {
                const int u = lane + 32 * k;
                const int qq = u < 8 * UPC ? u / UPC : 0;
                u_src[k] = __shfl_sync(0xFFFFFFFFu, src, 4 * qq);
                u_bytes[k] = __shfl_sync(0xFFFFFFFFu, bytes, 4 * qq);
            }
            for (uint32_t sf = 0; sf < nsl; ++sf) {
                if (!first) mbar_wait_s(empty_s + 8 * st, ph);
                const uint32_t dst = wring_s + st * WSTAGE;
#pragma unroll
                for (int k = 0; k < UPL; ++k) {
                    const int u = lane + 32 * k;
                    if (u < 8 * UPC) {
                        const int qq = u / UPC, off = (u % UPC) * 16;
                        const uint32_t g_off = sf * SL + off;
                        if (g_off < u_bytes[k]) {
                            KC_DCHECK(dst + qq * PITCH + swz_off(CFG::kSwz, qq, off) + 16 <=
                                      smem_u32(smem) + CFG::kRing);
                            KC_DCHECK(g_off + 16 <= u_bytes[k]);
                            cp_async16_s(dst + qq * PITCH + swz_off(CFG::kSwz, qq, off),
                                         reinterpret_cast<const uint8_t*>(u_src[k]) + g_off);
                        }
                    }
                }
                cp_async_mbar_arrive_noinc_s(full_s + 8 * st);
                if (++st == STAGES) { st = 0; ph ^= first ? 0u : 1u; first = false; }
            }
        }
        cp_async_wait<0>();
        return;
    }

    const unsigned qmask = 0xFu << (lane & 28);
    // shared addresses computed once: this lane's word of stage 0, the stage's barriers
    const uint64_t* xp0 = reinterpret_cast<const uint64_t*>(wring + q * PITCH) + ql;
    const int sq = CFG::kSwz ? (q & 3) : 0;  // stripe t of this quad at row position t ^ sq
    const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty);
    uint32_t st = 0, ph = 0;
    for (uint64_t j = j0; j < ngroups; j += W) {
        const uint64_t g = chunk_at(8 * j + q);
        ChunkRef cr = {nullptr, 0};
        if (g < C) cr = chunk_ref(regs, nreg, g, map);
        const uint32_t nst = cr.len >= 32 ? cr.len / 32 : 0;
        const uint32_t nsl = __reduce_max_sync(0xFFFFFFFFu, (nst * 32 + SL - 1) / SL);
        uint64_t v = lane_yseed(ql);  // y form
        uint32_t left = nst;  // this lane's stripes still to hash
        for (uint32_t s = 0; s < nsl; ++s) {
            mbar_wait_s(full_s + 8 * st, ph);
            const uint64_t* xp = xp0 + st * (WSTAGE / 8);
            KC_DCHECK(st < (uint32_t)STAGES &&
                      reinterpret_cast<const uint8_t*>(xp) - smem + 32 * (SL / 32 - 1) + 8 <= (long)CFG::kRing);
            if (left >= (uint32_t)(SL / 32)) {
                constexpr int UR = SL / 32 < 64 ? SL / 32 : 64;  // rounds unrolled per block (i-cache)
#pragma unroll 1
                for (int b = 0; b < SL / 32; b += UR) {
                    const uint64_t* xb = xp + 4 * b;
                    const uint64_t* pb[4] = {xb + 4 * (0 ^ sq), xb + 4 * (1 ^ sq), xb + 4 * (2 ^ sq), xb + 4 * (3 ^ sq)};
#pragma unroll
                    for (int t = 0; t < UR; ++t) v = ystep(v, pb[t & 3][4 * (t & ~3)]);
                }
                left -= SL / 32;
            } else {
                for (uint32_t t = 0; t < left; ++t) v = ystep(v, xp[4 * (t ^ sq)]);
                left = 0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_s(empty_s + 8 * st);
            if (++st == STAGES) { st = 0; ph ^= 1; }
        }
        if (g < C) {
            const uint64_t h = quad_finish<true>(yfinal(v), ql, qmask, cr.len, cr.src + (size_t)nst * 32);
            if (ql == 0) out[g] = h;
        } else {
            quad_finish<true>(yfinal(v), ql, qmask, 0, nullptr);
        }
    }
}

// ========================================================================== //
// K5 (F2 fused hash + compare): K1's cp.async ring staging BOTH the actual    //
// and the reference slice of 8 chunks per warp; each quad lane hashes its     //
// actual words (the post-manifest, bit-identical to K1) and ORs act ^ ref and //
// the reference's Inf/NaN exponent flags (float dtypes) into per-lane flags.  //
// A chunk is CLEAN when every bit agrees and the reference holds no Inf/NaN:  //
// it then contributes nothing to any report field, and K2 skips it.  Chunks   //
// with a sub-32-byte tail are marked dirty (K2 decides them exactly).         //
// ========================================================================== //
template <int WARPS, int STAGES, int SL>
struct CmpCfg {
    static constexpr int kWarps = WARPS, kStages = STAGES, kSlice = SL;
    static constexpr bool kSwz = true;
    static constexpr int kPitch = SL;  // swizzled rows (swz_off)
    static constexpr int kWStage = 16 * kPitch;          // 8 actual + 8 reference slices
    static constexpr int kUPC = SL / 16;                 // 16-byte units per slice
    static constexpr int kUPL = (16 * kUPC + 31) / 32;   // units per lane per step
    static constexpr size_t kSmem = (size_t)WARPS * STAGES * kWStage;
};

// special-exponent masks per dtype on the low / high 32-bit word of 8 bytes:
// ((w & M) + A) has bit H set exactly where an element's exponent is all ones
struct SpecMask { uint32_t m_lo, a_lo, m_hi, a_hi, h_lo, h_hi; };
__device__ __forceinline__ SpecMask spec_mask(int dt) {
    switch (dt) {
        case KC_DT_F16: return {0x7C007C00u, 0x04000400u, 0x7C007C00u, 0x04000400u, 0x80008000u, 0x80008000u};
        case KC_DT_BF16: return {0x7F807F80u, 0x00800080u, 0x7F807F80u, 0x00800080u, 0x80008000u, 0x80008000u};
        case KC_DT_F32: return {0x7F800000u, 0x00800000u, 0x7F800000u, 0x00800000u, 0x80000000u, 0x80000000u};
        case KC_DT_F64: return {0u, 0u, 0x7FF00000u, 0x00100000u, 0u, 0x80000000u};
        default: return {0u, 0u, 0u, 0u, 0u, 0u};
    }
}

// SELF (every pair has ref == act): only the actual slices are staged and the
// reference words are the actual ones, so one read gives the manifest and the
// Inf/NaN chunk flags (the host-reference validation's pass, kc_validate_host_ref)
template <class CFG, bool SELF = false>
__global__ void __launch_bounds__(CFG::kWarps * 32, 1)
    k5_hash_cmp(const PairDev* __restrict__ pairs, int npair, uint64_t C, uint64_t* __restrict__ out,
                unsigned long long* __restrict__ dirty, const uint32_t* __restrict__ map) {
    constexpr int WARPS = CFG::kWarps, STAGES = CFG::kStages, SL = CFG::kSlice, PITCH = CFG::kPitch;
    constexpr int WSTAGE = CFG::kWStage, UPC = CFG::kUPC, UPL = CFG::kUPL;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, q = lane >> 2, ql = lane & 3;
    const unsigned qmask = 0xFu << (lane & 28);
    uint8_t* wring = smem + (size_t)w * STAGES * WSTAGE;
    const uint32_t wring_s = smem_u32(wring);
    const uint64_t ngroups = (C + 7) / 8;
    const uint64_t W = (uint64_t)gridDim.x * WARPS;
    const uint64_t j0 = (uint64_t)w * gridDim.x + blockIdx.x;
    auto pair_of = [&](uint64_t g) -> int {
        if (map) return (int)__ldg(map + g);
        int lo = 0, hi = npair;  // last pair with chunk_off <= g
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pairs[mid].chunk_off <= g) lo = mid; else hi = mid;
        }
        return lo;
    };

    uint64_t jf = j0;
    uint32_t sf = 0, f_nsl = 0;
    unsigned long long u_src[UPL];
    uint32_t u_bytes[UPL];
    auto load_group = [&](uint64_t j) {
        const uint64_t g = 8 * j + q;
        unsigned long long sa = 0, sr = 0;
        uint32_t bytes = 0;
        if (g < C) {
            const PairDev& P = pairs[pair_of(g)];
            const uint64_t off = (g - P.chunk_off) * kChunk, rem = P.size - off;
            const uint32_t len = rem < kChunk ? (uint32_t)rem : (uint32_t)kChunk;
            sa = P.act + off;
            sr = P.ref + off;
            bytes = len >= 32 ? (len & ~31u) : 0u;
        }
        f_nsl = __reduce_max_sync(0xFFFFFFFFu, (bytes + SL - 1) / SL);
#pragma unroll
        for (int k = 0; k < UPL; ++k) {
            const int u = lane + 32 * k;
            const int qq = (u / UPC) & 7;
            const unsigned long long a = __shfl_sync(0xFFFFFFFFu, sa, 4 * qq);
            const unsigned long long r = __shfl_sync(0xFFFFFFFFu, sr, 4 * qq);
            u_src[k] = u < 8 * UPC ? a : r;
            u_bytes[k] = __shfl_sync(0xFFFFFFFFu, bytes, 4 * qq);
        }
    };
    auto issue = [&](int stage) {
        const uint32_t dst = wring_s + stage * WSTAGE;
#pragma unroll
        for (int k = 0; k < UPL; ++k) {
            const int u = lane + 32 * k;
            if (u < (SELF ? 8 : 16) * UPC) {
                const int slot = u / UPC, off = (u % UPC) * 16;  // slot 0-7 actual, 8-15 reference
                const uint32_t g_off = sf * SL + off;
                if (g_off < u_bytes[k]) {
                    KC_DCHECK(dst + slot * PITCH + swz_off(CFG::kSwz, slot, off) + 16 <=
                              wring_s - w * STAGES * WSTAGE + CFG::kSmem);
                    KC_DCHECK(g_off + 16 <= u_bytes[k]);
                    cp_async16_s(dst + slot * PITCH + swz_off(CFG::kSwz, slot, off),
                                 reinterpret_cast<const uint8_t*>(u_src[k]) + g_off);
                }
            }
        }
    };
    auto advance = [&]() {
        if (++sf >= f_nsl) {
            sf = 0;
            jf += W;
            if (jf < ngroups) load_group(jf); else f_nsl = 0;
        }
    };
    auto fetch = [&](int stage) {
        while (jf < ngroups && f_nsl == 0) {
            jf += W;
            if (jf < ngroups) load_group(jf);
        }
        if (jf < ngroups) {
            issue(stage);
            advance();
        }
        cp_async_commit();
    };
    if (j0 < ngroups) load_group(jf);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) fetch(s);
    uint32_t step = 0;
    for (uint64_t j = j0; j < ngroups; j += W) {
        const uint64_t g = 8 * j + q;
        const uint8_t* src = nullptr;
        uint32_t len = 0;
        SpecMask sm = {0u, 0u, 0u, 0u, 0u, 0u};
        if (g < C) {
            const PairDev& P = pairs[pair_of(g)];
            const uint64_t off = (g - P.chunk_off) * kChunk, rem = P.size - off;
            len = rem < kChunk ? (uint32_t)rem : (uint32_t)kChunk;
            src = reinterpret_cast<const uint8_t*>(P.act + off);
            sm = spec_mask(P.dtype);
        }
        const uint32_t nst = len >= 32 ? len / 32 : 0;
        const uint32_t nsl = __reduce_max_sync(0xFFFFFFFFu, (nst * 32 + SL - 1) / SL);
        uint64_t v = lane_yseed(ql);  // y form
        unsigned long long x = 0;
        uint32_t sp_lo = 0, sp_hi = 0;
        for (uint32_t s = 0; s < nsl; ++s, ++step) {
            cp_async_wait<STAGES - 2>();
            __syncwarp();
            const int st = step % STAGES;
            const uint64_t* pa = reinterpret_cast<const uint64_t*>(wring + st * WSTAGE + q * PITCH) + ql;
            const uint64_t* pr = reinterpret_cast<const uint64_t*>(wring + st * WSTAGE + (8 + q) * PITCH) + ql;
            const uint32_t done = s * (SL / 32);
            const uint32_t n = nst > done ? min((uint32_t)(SL / 32), nst - done) : 0u;
            const int sq = CFG::kSwz ? (q & 3) : 0;  // stripe t of this quad at row position t ^ sq
            auto word = [&](uint64_t a, uint64_t r) {
                v = ystep(v, a);
                if (!SELF) x |= a ^ r;
                sp_lo |= ((uint32_t)r & sm.m_lo) + sm.a_lo;
                sp_hi |= ((uint32_t)(r >> 32) & sm.m_hi) + sm.a_hi;
            };
            KC_DCHECK(reinterpret_cast<const uint8_t*>(pr) - smem + 32 * (SL / 32 - 1) + 8 <= (long)CFG::kSmem);
            if (n == SL / 32) {
                const int o[4] = {4 * (0 ^ sq), 4 * (1 ^ sq), 4 * (2 ^ sq), 4 * (3 ^ sq)};
#pragma unroll
                for (int t = 0; t < SL / 32; ++t) {
                    const uint64_t a = pa[o[t & 3] + 4 * (t & ~3)];
                    word(a, SELF ? a : pr[o[t & 3] + 4 * (t & ~3)]);
                }
            } else {
                for (uint32_t t = 0; t < n; ++t) {
                    const uint64_t a = pa[4 * (t ^ sq)];
                    word(a, SELF ? a : pr[4 * (t ^ sq)]);
                }
            }
            __syncwarp();
            fetch((step + STAGES - 1) % STAGES);
        }
        const bool mine = x != 0 || ((sp_lo & sm.h_lo) | (sp_hi & sm.h_hi)) != 0 || (len & 31u) != 0;
        const bool d = __ballot_sync(0xFFFFFFFFu, mine) & qmask;
        if (g < C) {
            const uint64_t h = quad_finish<true>(yfinal(v), ql, qmask, len, src + (size_t)nst * 32);
            if (ql == 0) {
                out[g] = h;
                if (d) atomicOr(dirty + (g >> 6), 1ULL << (g & 63));
            }
        } else {
            quad_finish<true>(yfinal(v), ql, qmask, 0, nullptr);
        }
    }
    cp_async_wait<0>();
}

// Unaligned regions (base % 16 != 0): quad per chunk, byte-assembled loads.
__global__ void __launch_bounds__(256)
    k1_hash_generic(const RegionDev* __restrict__ regs, int nreg, uint64_t C, uint64_t* __restrict__ out,
                    const uint32_t* __restrict__ map) {
    const int ql = threadIdx.x & 3;
    const unsigned qmask = 0xFu << (threadIdx.x & 28);
    const uint64_t nq = (uint64_t)gridDim.x * (blockDim.x / 4);
    for (uint64_t g = (uint64_t)blockIdx.x * (blockDim.x / 4) + (threadIdx.x >> 2); g < C; g += nq) {
        const ChunkRef cr = chunk_ref(regs, nreg, g, map);
        const uint64_t h = quad_xxh64_global<false>(cr.src, cr.len, ql, qmask);
        if (ql == 0) out[g] = h;
    }
}

// Region digests + the (base,size,digest) LE triples.  One warp per region
// streams the region's manifest (8 B per chunk, only 8-byte aligned) through a
// 2-stage shared-memory ring with 8-byte cp.async while lanes 0-3 (one quad)
// run the serial XXH64 chain from shared memory, so load latency is hidden
// behind the chain (~2,640 stripes for a 692 MB region).
constexpr int DG_STAGE = 8192;  // bytes per stage (multiple of 32)

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}

__global__ void __launch_bounds__(32)
    k1_region_digest(const RegionDev* __restrict__ regs, int nreg, const uint64_t* __restrict__ h,
                     uint64_t* __restrict__ dig, uint8_t* __restrict__ scratch) {
    __shared__ __align__(16) uint8_t buf[2][DG_STAGE];
    const int lane = threadIdx.x & 31, ql = lane & 3;
    for (int r = blockIdx.x; r < nreg; r += gridDim.x) {
        const uint64_t nck = (regs[r].size + kChunk - 1) / kChunk;
        const uint64_t len = 8 * nck;
        const uint8_t* p = reinterpret_cast<const uint8_t*>(h + regs[r].chunk_off);
        const uint64_t nst = len >= 32 ? len / 32 : 0;
        const uint64_t body = nst * 32;  // bytes consumed as stripes
        const uint32_t nstage = (uint32_t)((body + DG_STAGE - 1) / DG_STAGE);
        auto issue = [&](uint32_t k) {
            const uint64_t off = (uint64_t)k * DG_STAGE;
            const uint32_t b = (uint32_t)min((uint64_t)DG_STAGE, body - off);
            for (uint32_t o = 8 * lane; o < b; o += 256) cp_async8(&buf[k & 1][o], p + off + o);
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        uint64_t v = lane_yseed(ql);  // y form
        if (nstage > 0) issue(0);
        for (uint32_t k = 0; k < nstage; ++k) {
            if (k + 1 < nstage) {
                issue(k + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncwarp();
            if (lane < 4) {
                const uint64_t off = (uint64_t)k * DG_STAGE;
                const uint32_t n = (uint32_t)(min((uint64_t)DG_STAGE, body - off) / 32);
                const uint64_t* q = reinterpret_cast<const uint64_t*>(buf[k & 1]) + ql;
                uint32_t t = 0;
                for (; t + 8 <= n; t += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) v = ystep(v, q[4 * (t + u)]);
                }
                for (; t < n; ++t) v = ystep(v, q[4 * t]);
            }
            __syncwarp();  // stage k & 1 is rewritten by issue(k + 2)
        }
        if (lane < 4) {
            const uint64_t d = quad_finish<true>(yfinal(v), ql, 0xFu, len, p + body);
            if (lane == 0) {
                if (dig) dig[r] = d;
                if (scratch) {
                    uint64_t* t = reinterpret_cast<uint64_t*>(scratch + 24 * (size_t)r);
                    t[0] = regs[r].base;
                    t[1] = regs[r].size;
                    t[2] = d;
                }
            }
        }
        __syncwarp();
    }
}

__global__ void k1_snapshot_digest(const uint8_t* __restrict__ scratch, int nreg, uint64_t* __restrict__ out) {
    const int ql = threadIdx.x & 3;
    const uint64_t s = quad_xxh64_global<true>(scratch, 24 * (uint64_t)nreg, ql, 0xFu);
    if (threadIdx.x == 0) *out = s;
}

// ========================================================================== //
// K3: written set W[k] = (pre[k] != post[k]); warp per 64 chunks (ballots).  //
// ========================================================================== //
__global__ void k3_written(const uint64_t* __restrict__ pre, const uint64_t* __restrict__ post, uint64_t C,
                           uint64_t* __restrict__ bitmap, unsigned long long* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    const uint64_t nwords = (C + 63) / 64;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
    unsigned long long local = 0;
    for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); w < nwords; w += nwarps) {
        const uint64_t k0 = 64 * w + lane, k1 = k0 + 32;
        const bool b0 = k0 < C && __ldg(pre + k0) != __ldg(post + k0);
        const bool b1 = k1 < C && __ldg(pre + k1) != __ldg(post + k1);
        const uint32_t lo = __ballot_sync(0xFFFFFFFFu, b0);
        const uint32_t hi = __ballot_sync(0xFFFFFFFFu, b1);
        if (lane == 0) {
            bitmap[w] = (uint64_t)lo | ((uint64_t)hi << 32);
            local += __popc(lo) + __popc(hi);
        }
    }
    if (lane == 0 && local) atomicAdd(count, local);
}

// ========================================================================== //
// K2: fused diff.  Work = 16 KiB units of every segment, distributed to warps //
// in contiguous blocks.  Each lane streams 32-byte vectors of ref and act     //
// with 256-bit non-allocating loads (4 vectors of each in flight); equal      //
// vectors with no Inf/NaN exponent take the fast path.  Per-warp accumulators //
// flush with one atomic per nonzero field when the segment changes.          //
// ========================================================================== //
// Per-lane accumulators.  Counters are 32-bit: a warp flushes at least every
// kFlushUnits units (1 GiB), so one lane counts < 2^25 bytes between flushes.
struct Acc {
    uint32_t dbytes, delems, nan_r, nan_a, nan_pos, rel_undef, fail;
    unsigned long long max_ulp;
    double max_abs, max_rel;
    uint32_t any;  // this lane saw a differing byte in the current unit
    // 16-bit float fast path (elem16): an fp32 running max of exact |a - r|
    // (merged into max_abs at flush), RD32 of a value <= max_rel, and directed
    // fp32 roundings of atol / rtol (set once per launch, not by acc_zero)
    float mabs32, mrel32;
    float alo, ahi, rlo, rhi;
    uint32_t mulp16;  // running max ULP of the 16-bit common path (merged into max_ulp at flush)
};
constexpr uint64_t kFlushUnits = 65536;

__device__ __forceinline__ void acc_zero(Acc& a) {
    a.dbytes = a.delems = a.nan_r = a.nan_a = a.nan_pos = a.rel_undef = a.fail = a.max_ulp = 0;
    a.max_abs = 0.0;
    a.max_rel = 0.0;
    a.any = 0;
    a.mabs32 = a.mrel32 = 0.f;
    a.mulp16 = 0;
}

// number of nonzero bytes of x
__device__ __forceinline__ uint32_t nz_bytes(uint32_t x) {
    return __popc((((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u);
}

template <int DT> struct DT_;
template <> struct DT_<KC_DT_F16> { static constexpr int S = 2; static constexpr bool F = true; };
template <> struct DT_<KC_DT_BF16> { static constexpr int S = 2; static constexpr bool F = true; };
template <> struct DT_<KC_DT_F32> { static constexpr int S = 4; static constexpr bool F = true; };
template <> struct DT_<KC_DT_F64> { static constexpr int S = 8; static constexpr bool F = true; };
template <> struct DT_<KC_DT_BYTES> { static constexpr int S = 1; static constexpr bool F = false; };
template <> struct DT_<KC_DT_U8> { static constexpr int S = 1; static constexpr bool F = false; };
template <> struct DT_<KC_DT_I8> { static constexpr int S = 1; static constexpr bool F = false; };
template <> struct DT_<KC_DT_U16> { static constexpr int S = 2; static constexpr bool F = false; };
template <> struct DT_<KC_DT_I16> { static constexpr int S = 2; static constexpr bool F = false; };
template <> struct DT_<KC_DT_U32> { static constexpr int S = 4; static constexpr bool F = false; };
template <> struct DT_<KC_DT_I32> { static constexpr int S = 4; static constexpr bool F = false; };
template <> struct DT_<KC_DT_U64> { static constexpr int S = 8; static constexpr bool F = false; };
template <> struct DT_<KC_DT_I64> { static constexpr int S = 8; static constexpr bool F = false; };

template <int DT>
__device__ __forceinline__ bool is_signed_dt() {
    return DT == KC_DT_I8 || DT == KC_DT_I16 || DT == KC_DT_I32 || DT == KC_DT_I64;
}

// "exponent all ones" (Inf or NaN) anywhere in a 32-bit word of this dtype
template <int DT>
__device__ __forceinline__ uint32_t special_word(uint32_t w) {
    if (DT == KC_DT_F16) return ((w & 0x7C007C00u) + 0x04000400u) & 0x80008000u;
    if (DT == KC_DT_BF16) return ((w & 0x7F807F80u) + 0x00800080u) & 0x80008000u;
    if (DT == KC_DT_F32) return ((w & 0x7F800000u) + 0x00800000u) & 0x80000000u;
    if (DT == KC_DT_F64) return ((w & 0x7FF00000u) + 0x00100000u) & 0x80000000u;  // applied to hi words only
    return 0;
}

template <int DT, typename B>
__device__ __forceinline__ bool isnan_bits(B b) {
    if (DT == KC_DT_F16) return (b & 0x7FFFu) > 0x7C00u;
    if (DT == KC_DT_BF16) return (b & 0x7FFFu) > 0x7F80u;
    if (DT == KC_DT_F32) return (b & 0x7FFFFFFFu) > 0x7F800000u;
    return (b & 0x7FFFFFFFFFFFFFFFULL) > 0x7FF0000000000000ULL;
}

// exact conversion to fp64 (no FTZ: compiled without fast-math)
template <int DT, typename B>
__device__ __forceinline__ double to_f64(B b) {
    if (DT == KC_DT_F16) return (double)__half2float(__ushort_as_half((unsigned short)b));
    if (DT == KC_DT_BF16) return (double)__uint_as_float((uint32_t)b << 16);
    if (DT == KC_DT_F32) return (double)__uint_as_float((uint32_t)b);
    return __longlong_as_double((long long)b);
}

// One element (float dtypes): r, a raw bits (32-bit arithmetic below 8-byte types).
template <int DT>
__device__ __forceinline__ void elem_float(typename std::conditional<DT_<DT>::S == 8, uint64_t, uint32_t>::type r,
                                           typename std::conditional<DT_<DT>::S == 8, uint64_t, uint32_t>::type a,
                                           Acc& acc, double atol, double rtol, int equal_nan) {
    constexpr int S = DT_<DT>::S;
    using B = typename std::conditional<S == 8, uint64_t, uint32_t>::type;
    using SI = typename std::conditional<S == 8, long long, int>::type;
    const bool nr = isnan_bits<DT>(r), na = isnan_bits<DT>(a);
    const bool differ = r != a;
    acc.delems += differ;
    acc.nan_r += nr;
    acc.nan_a += na;
    acc.nan_pos += (nr != na);
    if (nr || na) {
        acc.fail += !(equal_nan && nr && na);
        return;
    }
    if (!differ) return;
    // ordered-integer ULP distance (|oa - orr| < 2^(8S), exact in B)
    const B sign = (B)1 << (8 * S - 1);
    const SI oa = (a & sign) ? -(SI)(a & ~sign) : (SI)a;
    const SI orr = (r & sign) ? -(SI)(r & ~sign) : (SI)r;
    const B ulp = oa >= orr ? (B)oa - (B)orr : (B)orr - (B)oa;
    if (ulp > acc.max_ulp) acc.max_ulp = ulp;
    const double av = to_f64<DT>(a), rv = to_f64<DT>(r);
    const double d = fabs(__dsub_rn(av, rv));
    if (d > acc.max_abs) acc.max_abs = d;
    const double ar = fabs(rv);
    const bool rfin = ar != CUDART_INF;
    // numpy.isclose(a, r) on fp64 (R27).  d <= atol already implies
    // d <= RN(atol + RN(rtol*|r|)) for rtol >= 0, so the product is skipped.
    bool close = (av == rv);
    if (!close && rfin) close = (d <= atol) || (d <= __dadd_rn(atol, __dmul_rn(rtol, ar)));
    acc.fail += !close;
    if (d != 0.0) {
        if (rv == 0.0) {
            acc.rel_undef += 1;
        } else if (!rfin) {
            acc.max_rel = CUDART_INF;
        } else if (d > __dmul_rd(acc.max_rel, ar)) {
            // only then can RN(d/|r|) exceed the running max: d <= RD(M*|r|) <= M*|r|
            // implies d/|r| <= M, and RN is monotonic
            const double rel = __ddiv_rn(d, ar);
            if (rel > acc.max_rel) acc.max_rel = rel;
        }
    }
}

// ---- 16-bit floats, fp32 fast path (DESIGN.md §7 K2, "16-bit fp32 path").  For finite f16/bf16 values
// whose exponent fields differ by at most KMAX, a - r is an integer below 2^24
// times a power of two inside fp32's range, so __fsub_rn returns it exactly and
// |a - r| equals the fp64 difference the oracle takes.  The two decisions
// that need fp64 are bracketed in fp32 with directed rounding:
//   isclose: L = RD(alo + RD(rlo*|r|)) <= RN64(atol + RN64(rtol*|r|)) <= U = RU(ahi + RU(rhi*|r|)),
//            so d <= L (or d <= alo) means close, d > U (and d > ahi) means not
//            close; in between the fp64 formula decides;
//   max_rel: d <= RD(mrel32*|r|) <= max_rel*|r| means RN64(d/|r|) <= max_rel, so
//            the fp64 division runs only when it can raise the running max.
// Everything else (Inf/NaN, exponents far apart, bf16 near overflow, equal bits
// with a special reference) takes elem_float unchanged.
#ifndef KC_K2_FAST16
#define KC_K2_FAST16 1
#endif
template <int DT>
__device__ __forceinline__ float f16bits_to_f32(uint32_t b) {
    if (DT == KC_DT_F16) return __half2float(__ushort_as_half((unsigned short)b));
    return __uint_as_float(b << 16);
}

template <int DT>
__device__ __forceinline__ void elem16(uint32_t r, uint32_t a, Acc& acc, double atol, double rtol, int equal_nan) {
    if constexpr (!KC_K2_FAST16) {
        elem_float<DT>(r, a, acc, atol, rtol, equal_nan);
        return;
    } else {
        constexpr int EB = DT == KC_DT_F16 ? 10 : 7;               // exponent field position
        constexpr uint32_t EM = DT == KC_DT_F16 ? 0x1Fu : 0xFFu;    // field mask
        constexpr uint32_t EFAST = DT == KC_DT_F16 ? 0x1Eu : 0xFDu; // largest field on the fast path
        constexpr uint32_t KMAX = DT == KC_DT_F16 ? 13u : 16u;      // (2^11-1)(2^13+1), (2^8-1)(2^16+1) < 2^24
        const uint32_t er = (r >> EB) & EM, ea = (a >> EB) & EM;
        const uint32_t de = er > ea ? er - ea : ea - er;  // raw fields: subnormals count one too far (conservative)
        if (er > EFAST || ea > EFAST || de > KMAX || r == a) {
            elem_float<DT>(r, a, acc, atol, rtol, equal_nan);
            return;
        }
        acc.delems += 1;
        const int oa = (a & 0x8000u) ? -(int)(a & 0x7FFFu) : (int)a;
        const int orr = (r & 0x8000u) ? -(int)(r & 0x7FFFu) : (int)r;
        const unsigned long long ulp = (unsigned long long)(oa >= orr ? oa - orr : orr - oa);
        if (ulp > acc.max_ulp) acc.max_ulp = ulp;
        const float av = f16bits_to_f32<DT>(a), rv = f16bits_to_f32<DT>(r);
        const float d = fabsf(__fsub_rn(av, rv));  // exact
        acc.mabs32 = fmaxf(acc.mabs32, d);
        if (d == 0.f) return;  // +0 vs -0: close, no relative error
        const float ar = fabsf(rv);
        bool close;
        if (d <= acc.alo || d <= __fadd_rd(acc.alo, __fmul_rd(acc.rlo, ar))) {
            close = true;
        } else if (d > acc.ahi && d > __fadd_ru(acc.ahi, __fmul_ru(acc.rhi, ar))) {
            close = false;
        } else {
            const double dd = (double)d;
            close = (dd <= atol) || (dd <= __dadd_rn(atol, __dmul_rn(rtol, (double)ar)));
        }
        acc.fail += !close;
        if (rv == 0.f) {
            acc.rel_undef += 1;
        } else if (d > __fmul_rd(acc.mrel32, ar)) {
            const double rel = __ddiv_rn((double)d, (double)ar);
            if (rel > acc.max_rel) {
                acc.max_rel = rel;
                acc.mrel32 = __double2float_rd(rel);
            }
        }
    }
}

// ---- 16-bit common case, branch-free (the drain rounds of the element queue).
// An element is handled here, with exactly elem16's result, when it is a
// same-sign pair of finite nonzero values whose magnitudes are within a factor
// 2^KMAX of each other (so their exponents differ by at most KMAX, 13 for f16
// and 16 for bf16, and a - r is exact in fp32: |a - r| <= max(|a|, |r|) is an
// integer below (2^p - 1)(2^KMAX + 1) < 2^24 times the smaller ulp, and same
// signs cannot overflow), that differ (d != 0), whose isclose decision lies
// outside the directed-rounding bracket, and which cannot raise the running
// max_rel (d <= RD(mrel32 * |r|)).  Then: delems += 1, ULP = |bits(a) - bits(r)|
// (same sign), |a - r| into the fp32 max, fail += !close.  Anything else
// (Inf/NaN, zeros, far exponents, opposite signs, equal bits, an ambiguous
// isclose, a max_rel candidate) returns true: the rare queue runs elem16 on it.
template <int DT>
__device__ __forceinline__ bool elem16_rare(uint32_t t, uint32_t xs, Acc& acc) {
    // tl / th: the reference / actual bits in the high half; xs = t ^ tl, whose high
    // half is a ^ r (bit 31: the signs differ); computed once by the caller
    const uint32_t tl = t << 16, th = t & 0xFFFF0000u;
    float av, rv;
    if constexpr (DT == KC_DT_BF16) {
        av = __uint_as_float(th);
        rv = __uint_as_float(tl);
    } else {
        av = __half2float(__ushort_as_half((unsigned short)(t >> 16)));
        rv = __half2float(__ushort_as_half((unsigned short)(t & 0xFFFFu)));
    }
    constexpr float RATIO = DT == KC_DT_F16 ? 8192.f : 65536.f;  // 2^KMAX
    const float d = fabsf(__fsub_rn(av, rv));
    const float ar = fabsf(rv), aa = fabsf(av);
    const bool close_lo = d <= __fadd_rd(acc.alo, __fmul_rd(acc.rlo, ar));
    const bool far_hi = d > __fadd_ru(acc.ahi, __fmul_ru(acc.rhi, ar));
    const bool common = (ar < __fmul_rn(RATIO, aa)) & (aa < __fmul_rn(RATIO, ar)) & ((int)xs >= 0) &
                        (d != 0.f) & (close_lo != far_hi) & (d <= __fmul_rd(acc.mrel32, ar));
    if (common) {
        acc.delems += 1;
        // same signs: |bits(a) - bits(r)| < 2^15, so (th - tl) = (a - r) * 2^16 fits an int
        acc.mulp16 = max(acc.mulp16, (uint32_t)abs((int)th - (int)tl) >> 16);
        acc.mabs32 = fmaxf(acc.mabs32, d);
        acc.fail += far_hi;
    }
    return !common;
}

template <int DT>
__device__ __forceinline__ void elem_int(uint64_t r, uint64_t a, Acc& acc) {
    constexpr int S = DT_<DT>::S;
    if (r == a) return;
    acc.delems += 1;
    unsigned long long d;
    if (is_signed_dt<DT>()) {
        const int sh = 64 - 8 * S;
        const long long va = (long long)(a << sh) >> sh, vr = (long long)(r << sh) >> sh;
        d = va >= vr ? (unsigned long long)va - (unsigned long long)vr : (unsigned long long)vr - (unsigned long long)va;
    } else {
        d = a >= r ? a - r : r - a;
    }
    if (d > acc.max_ulp) acc.max_ulp = d;
}

// select word i (0..7) of an 8-word register vector without local memory
__device__ __forceinline__ uint32_t sel8(const uint32_t (&w)[8], int i) {
    const uint32_t a = (i & 1) ? w[1] : w[0], b = (i & 1) ? w[3] : w[2];
    const uint32_t c = (i & 1) ? w[5] : w[4], d = (i & 1) ? w[7] : w[6];
    const uint32_t e = (i & 2) ? b : a, f = (i & 2) ? d : c;
    return (i & 4) ? f : e;
}

// Fast check of one 32-byte vector pair: counts differing bytes, and returns
// the mask of elements that need the per-element path (differing bits, or an
// Inf/NaN exponent on either side for float types).  BYTES is finished here.
template <int DT>
__device__ __forceinline__ uint32_t vec_scan(const uint32_t (&r)[8], const uint32_t (&a)[8], Acc& acc) {
    constexpr int S = DT_<DT>::S;
    constexpr bool F = DT_<DT>::F;
    uint32_t x[8];
    uint32_t anyx = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = r[i] ^ a[i];
        anyx |= x[i];
    }
    if (anyx == 0) {
        // bit-equal vector: only a NaN (counted, and failing allclose unless
        // equal_nan) can matter, and then special(a) == special(r)
        if (!F) return 0;
        uint32_t spec = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (S != 8 || (i & 1)) spec |= special_word<DT>(r[i]);
        if (spec == 0) return 0;  // fast path
    } else {
        acc.any = 1;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc.dbytes += nz_bytes(x[i]);
        if (DT == KC_DT_BYTES) {
            uint32_t m = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) m = __vmaxu4(m, __vabsdiffu4(r[i], a[i]));
            m = max(max(m & 0xFF, (m >> 8) & 0xFF), max((m >> 16) & 0xFF, m >> 24));
            if (m > acc.max_ulp) acc.max_ulp = m;
            return 0;
        }
    }
    // an element is flagged when its bits differ, or (float types) when the
    // reference is Inf/NaN: an element with equal bits has special(a) ==
    // special(r), and one with differing bits is flagged already
    uint32_t mask = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (S == 8) {
            if (i & 1) {
                const uint32_t sp = F ? special_word<DT>(r[i]) : 0u;
                mask |= (uint32_t)(((x[i - 1] | x[i]) | sp) != 0) << (i >> 1);
            }
        } else if (S == 4) {
            const uint32_t sp = F ? special_word<DT>(r[i]) : 0u;
            mask |= (uint32_t)((x[i] | sp) != 0) << i;
        } else if (S == 2) {
            uint32_t m = (((x[i] & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x[i]) & 0x80008000u;
            if (F) m |= special_word<DT>(r[i]);
            mask |= (((m >> 15) & 1u) | ((m >> 30) & 2u)) << (2 * i);
        } else {
            const uint32_t m = (((x[i] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x[i]) & 0x80808080u;
            mask |= (((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u)) << (4 * i);
        }
    }
    return mask;
}

// Per-element path for the elements in mask (one code copy: element bits are
// picked out of the register vector with selects).
template <int DT>
__device__ __forceinline__ void vec_slow(const uint32_t (&r)[8], const uint32_t (&a)[8], uint32_t mask, Acc& acc,
                                         double atol, double rtol, int equal_nan) {
    constexpr int S = DT_<DT>::S;
    while (mask) {
        const int e = __ffs(mask) - 1;
        mask &= mask - 1;
        uint64_t rb, ab;
        if (S == 8) {
            rb = (uint64_t)sel8(r, 2 * e) | ((uint64_t)sel8(r, 2 * e + 1) << 32);
            ab = (uint64_t)sel8(a, 2 * e) | ((uint64_t)sel8(a, 2 * e + 1) << 32);
        } else if (S == 4) {
            rb = sel8(r, e);
            ab = sel8(a, e);
        } else if (S == 2) {
            rb = (sel8(r, e >> 1) >> (16 * (e & 1))) & 0xFFFFu;
            ab = (sel8(a, e >> 1) >> (16 * (e & 1))) & 0xFFFFu;
        } else {
            rb = (sel8(r, e >> 2) >> (8 * (e & 3))) & 0xFFu;
            ab = (sel8(a, e >> 2) >> (8 * (e & 3))) & 0xFFu;
        }
        if (DT_<DT>::F) elem_float<DT>(rb, ab, acc, atol, rtol, equal_nan); else elem_int<DT>(rb, ab, acc);
    }
}

// ---- compacted per-element path for float dtypes: every lane appends the
// (ref, act) bits of its flagged elements to a per-warp shared-memory queue
// (warp prefix sum for the slots); full rounds of 32 elements are then
// processed with every lane busy, instead of each lane looping over its own
// mask (SIMT runs the longest lane's loop: ~12 of 32 lanes were active at
// 11% mismatch density).  All accumulations are sums and maxima, so the order
// in which elements are processed does not change a report bit.
#ifndef KC_GENERIC_SCAN16
#define KC_GENERIC_SCAN16 0  // 1: 16-bit floats through the generic packed-mask scan (comparison builds)
#endif
constexpr bool kGenericScan16 = KC_GENERIC_SCAN16 != 0;
template <int DT> struct QT_ { using T = uint32_t; };  // 2-byte types: r | a << 16
template <> struct QT_<KC_DT_F32> { using T = uint2; };
template <> struct QT_<KC_DT_F64> { using T = ulonglong2; };
template <int DT, int U>
struct KQ {  // queue capacity: < 32 carried + the most one step can append
    static constexpr int kCap = 32 + 32 * U * (32 / DT_<DT>::S);
    static constexpr int kBytes = kCap * (int)sizeof(typename QT_<DT>::T);
};

template <int DT>
__device__ __forceinline__ void q_push(const uint32_t (&r)[8], const uint32_t (&a)[8], uint32_t mask,
                                       typename QT_<DT>::T* q, uint32_t& pos) {
    constexpr int S = DT_<DT>::S;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if constexpr (S == 2) {
            if (mask & (1u << (2 * i))) q[pos++] = __byte_perm(r[i], a[i], 0x5410);
            if (mask & (2u << (2 * i))) q[pos++] = __byte_perm(r[i], a[i], 0x7632);
        } else if constexpr (S == 4) {
            if (mask & (1u << i)) q[pos++] = make_uint2(r[i], a[i]);
        } else {
            if ((i & 1) && (mask & (1u << (i >> 1))))
                q[pos++] = make_ulonglong2((unsigned long long)r[i - 1] | ((unsigned long long)r[i] << 32),
                                           (unsigned long long)a[i - 1] | ((unsigned long long)a[i] << 32));
        }
    }
}

// ---- 16-bit floats (the c3 case): the element flags stay as bits 15 / 31 of
// eight words per vector instead of a packed mask.  A half is flagged when its
// bits differ or the reference half has an all-ones exponent: both tests are
// "add a constant below the sign bit, look at bit 15 / 31", merged into one
// LOP3 per word.  The flagged halves are counted with IDP.4A and pushed by
// testing the word bits directly.  Differing bytes are not counted here: every
// element with a differing byte is flagged, so q_item counts its bytes.
template <int DT>
__device__ __forceinline__ uint32_t vec_scan16(const uint32_t (&r)[8], const uint32_t (&a)[8], uint32_t (&m)[8],
                                               uint32_t& cnt128, Acc& acc) {
    uint32_t x[8], anyx = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = r[i] ^ a[i];
        anyx |= x[i];
    }
    uint32_t any = 0;
    if (anyx == 0) {  // bit-equal vector: only Inf/NaN references need the element path
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            m[i] = special_word<DT>(r[i]);
            any |= m[i];
        }
    } else {
        acc.any = 1;
        constexpr uint32_t EX = DT == KC_DT_F16 ? 0x7C007C00u : 0x7F807F80u;
        constexpr uint32_t EI = DT == KC_DT_F16 ? 0x04000400u : 0x00800080u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t nz = ((x[i] & 0x7FFF7FFFu) + 0x7FFF7FFFu) | x[i];  // bit 15/31: half differs
            const uint32_t sp = (r[i] & EX) + EI;                               // bit 15/31: Inf/NaN ref
            m[i] = (nz | sp) & 0x80008000u;
            any |= m[i];
        }
    }
    if (any) {
#pragma unroll
        for (int i = 0; i < 8; ++i) cnt128 = __dp4a(m[i], 0x01010101u, cnt128);
    }
    return any;
}

// Round 2: the same flags with the half-precision compare unit doing most of
// the work (the ALU pipe binds the planted case, ncu: ALU 78%, FMA 20%).  A
// half needs the element path iff its bits differ or a side is NaN:
//   HSET2.NEU(r, a) is true for every pair of unequal values and for every NaN
//   (unordered), and false only for equal values; equal values with unequal
//   bits are exactly +0 / -0 (f16 and bf16 have no other duplicate encodings,
//   subnormals are compared as values: set.*.f16x2 / bf16x2 honour them), whose
//   sign bits differ.  So flag = NEU(r, a) | ((r ^ a) & sign): one HSET2 and
//   one LOP3 per word.  An Inf reference with equal bits contributes nothing to
//   any report field (elem_float returns at once), so it is no longer flagged.
// acc.any (a differing byte in this unit, for the bitmap) still needs the raw
// XOR, taken only for vectors with a flag.
template <int DT>
__device__ __forceinline__ uint32_t ne_mask16(uint32_t r, uint32_t a) {
    if constexpr (DT == KC_DT_F16) {
        return __hneu2_mask(*reinterpret_cast<const __half2*>(&r), *reinterpret_cast<const __half2*>(&a));
    } else {
        return __hneu2_mask(*reinterpret_cast<const __nv_bfloat162*>(&r),
                            *reinterpret_cast<const __nv_bfloat162*>(&a));
    }
}

template <int DT>
__device__ __forceinline__ uint32_t vec_scan16h(const uint32_t (&r)[8], const uint32_t (&a)[8], uint32_t (&m)[8],
                                                uint32_t& cnt128, Acc& acc) {
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        m[i] = (ne_mask16<DT>(r[i], a[i]) | (r[i] ^ a[i])) & 0x80008000u;
        any |= m[i];
    }
    if (any) {
        uint32_t anyx = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) anyx |= r[i] ^ a[i];
        acc.any |= (uint32_t)(anyx != 0);
#pragma unroll
        for (int i = 0; i < 8; ++i) cnt128 = __dp4a(m[i], 0x01010101u, cnt128);
    }
    return any;
}

template <int DT>
__device__ __forceinline__ void q_push16(const uint32_t (&r)[8], const uint32_t (&a)[8], const uint32_t (&m)[8],
                                         uint32_t* q, uint32_t& pos) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (m[i] & 0x00008000u) q[pos++] = __byte_perm(r[i], a[i], 0x5410);
        if (m[i] & 0x80000000u) q[pos++] = __byte_perm(r[i], a[i], 0x7632);
    }
}

// the same push as one shared-memory byte address bumped by the flag bits
// (no serial increment/move chain per element)
__device__ __forceinline__ void q_push16_addr(const uint32_t (&r)[8], const uint32_t (&a)[8], const uint32_t (&m)[8],
                                              uint32_t& sa) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (m[i] & 0x00008000u)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(__byte_perm(r[i], a[i], 0x5410)) : "memory");
        sa += (m[i] >> 13) & 4u;
        if (m[i] & 0x80000000u)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(__byte_perm(r[i], a[i], 0x7632)) : "memory");
        sa += (m[i] >> 29) & 4u;
    }
}

// Q2 = 3 push (default): one ALU op per address bump instead of three (the ALU
// pipe binds this path, ncu: ALU 79%).  m is masked to bits 15 / 31; f = m &
// 0x8000 (the LOP3 that also sets the store predicate) gives 4 * bit15 =
// hi32(f * 2^19) and 4 * bit31 = hi32(m * 8) (bit 15 does not reach), each a
// mad.hi.u32 by a power of two, which ptxas emits as one LEA.HI.  (The same
// bumps as IMAD.HI on the FMA pipe, with multipliers hidden from ptxas, were
// slower: a serial chain of 4-cycle IMADs, 5.2 vs 5.8 TB/s.)
__device__ __forceinline__ uint32_t bump_hi(uint32_t v, uint32_t mul, uint32_t sa) {
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(v), "r"(mul), "r"(sa));
    return d;
}
__device__ __forceinline__ void q_push16_lea(const uint32_t (&r)[8], const uint32_t (&a)[8], const uint32_t (&m)[8],
                                             uint32_t& sa) {
    constexpr uint32_t k19 = 1u << 19, k3 = 8u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t f = m[i] & 0x00008000u;
        if (f) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(__byte_perm(r[i], a[i], 0x5410)) : "memory");
        sa = bump_hi(f, k19, sa);
        if ((int)m[i] < 0)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(sa), "r"(__byte_perm(r[i], a[i], 0x7632)) : "memory");
        sa = bump_hi(m[i], k3, sa);
    }
}

template <int DT>
__device__ __forceinline__ void q_item(typename QT_<DT>::T t, Acc& acc, double atol, double rtol, int equal_nan) {
    if constexpr (DT_<DT>::S == 2) {
        if constexpr (!kGenericScan16) {  // vec_scan16 leaves the differing bytes to the element
            const uint32_t x = (t ^ (t >> 16)) & 0xFFFFu;
            acc.dbytes += (uint32_t)((x & 0xFFu) != 0) + (uint32_t)(x > 0xFFu);
        }
        elem16<DT>(t & 0xFFFFu, t >> 16, acc, atol, rtol, equal_nan);
    } else
        elem_float<DT>(t.x, t.y, acc, atol, rtol, equal_nan);
}

// process floor(qn/32) full rounds, move the remainder to the front
template <int DT>
__device__ __forceinline__ void q_drain(typename QT_<DT>::T* q, uint32_t& qn, Acc& acc, double atol, double rtol,
                                        int equal_nan, int lane) {
    __syncwarp();
    const uint32_t full = qn & ~31u, rem = qn - full;
    for (uint32_t i = lane; i < full; i += 32) q_item<DT>(q[i], acc, atol, rtol, equal_nan);
    typename QT_<DT>::T t;
    if (lane < rem) t = q[full + lane];
    __syncwarp();
    if (lane < rem) q[lane] = t;
    __syncwarp();
    qn = rem;
}

// process everything left (before a report flush)
template <int DT>
__device__ __forceinline__ void q_finish(typename QT_<DT>::T* q, uint32_t& qn, Acc& acc, double atol, double rtol,
                                         int equal_nan, int lane) {
    if constexpr (DT_<DT>::F) {
        if (qn == 0) return;
        __syncwarp();
        if (lane < qn) q_item<DT>(q[lane], acc, atol, rtol, equal_nan);
        __syncwarp();
        qn = 0;
    }
}

// 16-bit floats with the rare queue (Q2): each drain round runs the branch-free
// common case (elem16_rare) on 32 queued elements; the elements it declines are
// appended to a second per-warp queue (rq, < 64 entries, ballot slots) and
// processed 32 at a time by elem16 when that queue fills.  Every element is
// handled exactly once by exactly one of the two, so the report is unchanged.
constexpr int kRareBytes = 64 * 4;  // rare queue per warp

template <int DT>
__device__ __forceinline__ void rq_round(uint32_t* rq, uint32_t& rn, Acc& acc, double atol, double rtol,
                                         int equal_nan, int lane) {
    __syncwarp();
    const uint32_t t = rq[lane];
    elem16<DT>(t & 0xFFFFu, t >> 16, acc, atol, rtol, equal_nan);
    const uint32_t left = rn - 32;
    uint32_t u = 0;
    if (lane < left) u = rq[32 + lane];
    __syncwarp();
    if (lane < left) rq[lane] = u;
    __syncwarp();
    rn = left;
}

template <int DT>
__device__ __forceinline__ void q_drain16(uint32_t* q, uint32_t& qn, uint32_t* rq, uint32_t& rn, Acc& acc,
                                          double atol, double rtol, int equal_nan, int lane) {
    __syncwarp();
    const uint32_t full = qn & ~31u, rem = qn - full;
    uint32_t lt;  // lanes below this one (a special register: not re-derived inside the loop)
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (uint32_t i = lane; i < full; i += 32) {
        const uint32_t t = q[i];
        const uint32_t xs = t ^ (t << 16);  // high half: a ^ r; every queued element's bytes are counted here
        acc.dbytes += (uint32_t)((xs & 0x00FF0000u) != 0) + (uint32_t)(xs >= 0x01000000u);
        const bool rare = elem16_rare<DT>(t, xs, acc);
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, rare);
        KC_DCHECK(rn + __popc(bal) <= (uint32_t)(kRareBytes / 4));
        if (rare) rq[rn + __popc(bal & lt)] = t;
        rn += __popc(bal);
        if (rn >= 32) rq_round<DT>(rq, rn, acc, atol, rtol, equal_nan, lane);
    }
    uint32_t t = 0;
    if (lane < rem) t = q[full + lane];
    __syncwarp();
    if (lane < rem) q[lane] = t;
    __syncwarp();
    qn = rem;
}

// everything left in both queues (before a report flush)
template <int DT>
__device__ __forceinline__ void q_finish16(uint32_t* q, uint32_t& qn, uint32_t* rq, uint32_t& rn, Acc& acc,
                                           double atol, double rtol, int equal_nan, int lane) {
    if (qn) {
        __syncwarp();
        if (lane < qn) q_item<DT>(q[lane], acc, atol, rtol, equal_nan);
        qn = 0;
    }
    if (rn) {
        __syncwarp();
        if (lane < rn) elem16<DT>(rq[lane] & 0xFFFFu, rq[lane] >> 16, acc, atol, rtol, equal_nan);
        rn = 0;
    }
    __syncwarp();
}

// scalar path: one element at byte offset o (element-size aligned within the buffer)
template <int DT>
__device__ __forceinline__ void elem_scalar(const uint8_t* R, const uint8_t* A, Acc& acc, double atol, double rtol,
                                            int equal_nan) {
    constexpr int S = DT_<DT>::S;
    uint64_t rb = 0, ab = 0;
#pragma unroll
    for (int i = S - 1; i >= 0; --i) {
        rb = (rb << 8) | __ldg(R + i);
        ab = (ab << 8) | __ldg(A + i);
    }
    if (rb != ab) {
        acc.any = 1;
        uint64_t x = rb ^ ab;
#pragma unroll
        for (int i = 0; i < S; ++i) acc.dbytes += ((x >> (8 * i)) & 0xFF) != 0;
    }
    if (DT == KC_DT_BYTES) {
        const unsigned long long d = rb > ab ? rb - ab : ab - rb;
        if (d > acc.max_ulp) acc.max_ulp = d;
        return;
    }
    if (DT_<DT>::F) elem_float<DT>(rb, ab, acc, atol, rtol, equal_nan); else elem_int<DT>(rb, ab, acc);
}

__device__ __forceinline__ void ld256(const void* p, uint32_t* w) {
    unsigned long long a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
    w[0] = (uint32_t)a; w[1] = (uint32_t)(a >> 32);
    w[2] = (uint32_t)b; w[3] = (uint32_t)(b >> 32);
    w[4] = (uint32_t)c; w[5] = (uint32_t)(c >> 32);
    w[6] = (uint32_t)d; w[7] = (uint32_t)(d >> 32);
}

// one unit [off, off+len) of a segment, whole warp: U vectors of each stream
// in flight per lane; the per-element path runs once per vector that needs it.
template <int DT, int U, int Q2>
__device__ __forceinline__ void diff_unit(const uint8_t* R, const uint8_t* A, uint32_t len, bool vec_ok, Acc& acc,
                                          double atol, double rtol, int equal_nan, int lane,
                                          typename QT_<DT>::T* q, uint32_t& qn, uint32_t* rq, uint32_t& rn) {
    constexpr int S = DT_<DT>::S;
    uint32_t done = 0;
    if (vec_ok) {
        const uint32_t nvec = len / 32;
        uint32_t v = lane;
        if constexpr (DT_<DT>::F && S == 2 && !kGenericScan16 && Q2) {
            // 16-bit floats, software-pipelined: step k+1's vectors are loaded into
            // the registers step k's push has just finished with, BEFORE step k's
            // queue drain, so the drain's ALU work covers the load latency (ncu:
            // the first use of each step's loads was the top stall, ~27% of samples)
            const uint32_t nsteps = nvec / (32 * U);  // warp-uniform
            if (nsteps) {
                uint32_t rw[U][8], aw[U][8];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    ld256(R + 32 * (size_t)(v + 32 * u), rw[u]);
                    ld256(A + 32 * (size_t)(v + 32 * u), aw[u]);
                }
                for (uint32_t k = 0; k < nsteps; ++k) {
                    uint32_t mw[U][8];
                    uint32_t any = 0, cnt128 = 0;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        any |= Q2 >= 2 ? vec_scan16h<DT>(rw[u], aw[u], mw[u], cnt128, acc)
                                       : vec_scan16<DT>(rw[u], aw[u], mw[u], cnt128, acc);
                    const bool push = __any_sync(0xFFFFFFFFu, any != 0);
                    if (push) {
                        const uint32_t c = cnt128 >> 7;
                        uint32_t incl = c;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                            if (lane >= d) incl += t;
                        }
                        const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
                        uint32_t sa = (uint32_t)__cvta_generic_to_shared(q) + 4 * (qn + incl - c);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if constexpr (Q2 == 3) q_push16_lea(rw[u], aw[u], mw[u], sa);
                            else q_push16_addr(rw[u], aw[u], mw[u], sa);
                        }
                        qn += total;
                        KC_DCHECK((qn <= (uint32_t)KQ<DT, U>::kCap));
                    }
                    v += 32 * U;
                    if (k + 1 < nsteps) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            ld256(R + 32 * (size_t)(v + 32 * u), rw[u]);
                            ld256(A + 32 * (size_t)(v + 32 * u), aw[u]);
                        }
                    }
                    if (qn >= 32) q_drain16<DT>(q, qn, rq, rn, acc, atol, rtol, equal_nan, lane);
                }
            }
        }
        // every lane runs the same number of U-steps (nvec is warp-uniform), so
        // the warp-wide queue operations below see all 32 lanes
        for (; v - lane + 32 * U <= nvec; v += 32 * U) {
            uint32_t rw[U][8], aw[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                ld256(R + 32 * (size_t)(v + 32 * u), rw[u]);
                ld256(A + 32 * (size_t)(v + 32 * u), aw[u]);
            }
            if constexpr (DT_<DT>::F && S == 2 && !kGenericScan16) {
                uint32_t mw[U][8];
                uint32_t any = 0, cnt128 = 0;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    any |= Q2 >= 2 ? vec_scan16h<DT>(rw[u], aw[u], mw[u], cnt128, acc)
                                   : vec_scan16<DT>(rw[u], aw[u], mw[u], cnt128, acc);
                if (__any_sync(0xFFFFFFFFu, any != 0)) {
                    const uint32_t c = cnt128 >> 7;
                    uint32_t incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                        if (lane >= d) incl += t;
                    }
                    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
                    uint32_t pos = qn + incl - c;
                    if constexpr (Q2) {
                        uint32_t sa = (uint32_t)__cvta_generic_to_shared(q) + 4 * pos;
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if constexpr (Q2 == 3) q_push16_lea(rw[u], aw[u], mw[u], sa);
                            else q_push16_addr(rw[u], aw[u], mw[u], sa);
                        }
                        qn += total;
                        KC_DCHECK((qn <= (uint32_t)KQ<DT, U>::kCap));
                        if (qn >= 32) q_drain16<DT>(q, qn, rq, rn, acc, atol, rtol, equal_nan, lane);
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) q_push16<DT>(rw[u], aw[u], mw[u], q, pos);
                        qn += total;
                        KC_DCHECK((qn <= (uint32_t)KQ<DT, U>::kCap));
                        if (qn >= 32) q_drain<DT>(q, qn, acc, atol, rtol, equal_nan, lane);
                    }
                }
                continue;
            }
            uint32_t m[U];
            uint32_t any = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                m[u] = vec_scan<DT>(rw[u], aw[u], acc);
                any |= m[u];
            }
            if constexpr (DT_<DT>::F) {
                if (__any_sync(0xFFFFFFFFu, any != 0)) {
                    uint32_t c = 0;
#pragma unroll
                    for (int u = 0; u < U; ++u) c += __popc(m[u]);
                    uint32_t incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                        if (lane >= d) incl += t;
                    }
                    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
                    uint32_t pos = qn + incl - c;
#pragma unroll
                    for (int u = 0; u < U; ++u) q_push<DT>(rw[u], aw[u], m[u], q, pos);
                    qn += total;
                        KC_DCHECK((qn <= (uint32_t)KQ<DT, U>::kCap));
                    if (qn >= 32) q_drain<DT>(q, qn, acc, atol, rtol, equal_nan, lane);
                }
                continue;
            }
            if (any) {
#pragma unroll 1
                for (int u = 0; u < U; ++u) {
                    uint32_t mu = m[0];
#pragma unroll
                    for (int k = 1; k < U; ++k) mu = u == k ? m[k] : mu;
                    if (!mu) continue;
                    uint32_t rr[8], aa[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        rr[i] = rw[0][i];
                        aa[i] = aw[0][i];
#pragma unroll
                        for (int k = 1; k < U; ++k) {
                            rr[i] = u == k ? rw[k][i] : rr[i];
                            aa[i] = u == k ? aw[k][i] : aa[i];
                        }
                    }
                    vec_slow<DT>(rr, aa, mu, acc, atol, rtol, equal_nan);
                }
            }
        }
        for (; v < nvec; v += 32) {
            uint32_t r0[8], a0[8];
            ld256(R + 32 * (size_t)v, r0);
            ld256(A + 32 * (size_t)v, a0);
            const uint32_t m0 = vec_scan<DT>(r0, a0, acc);
            if (m0) vec_slow<DT>(r0, a0, m0, acc, atol, rtol, equal_nan);
        }
        done = nvec * 32;
    }
    for (uint32_t o = done + lane * S; o < len; o += 32 * S) elem_scalar<DT>(R + o, A + o, acc, atol, rtol, equal_nan);
}

// Warp reductions with the REDUX unit (one instruction each): 64-bit sums as
// two 32-bit partial sums (valid while every lane's value is < 2^48, i.e. for
// any segment < 256 TiB), 64-bit maxima as max of the high words, then of the
// low words among the lanes holding that high word.
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
    const uint32_t lo = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(v & 0xFFFFu));
    const uint32_t hi = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(v >> 16));
    return ((unsigned long long)hi << 16) + lo;
}
__device__ __forceinline__ unsigned long long warp_maxu(unsigned long long v) {
    const uint32_t hi = __reduce_max_sync(0xFFFFFFFFu, (uint32_t)(v >> 32));
    const uint32_t lo = __reduce_max_sync(0xFFFFFFFFu, (uint32_t)(v >> 32) == hi ? (uint32_t)v : 0u);
    return ((unsigned long long)hi << 32) | lo;
}

__device__ void acc_flush(Acc& acc, kc_diff_report* rep, int lane) {
    const unsigned FULL = 0xFFFFFFFFu;
    acc.max_abs = fmax(acc.max_abs, (double)acc.mabs32);  // both exact values
    if (acc.mulp16 > acc.max_ulp) acc.max_ulp = acc.mulp16;
    const unsigned long long mabs = (unsigned long long)__double_as_longlong(acc.max_abs);
    const unsigned long long mrel = (unsigned long long)__double_as_longlong(acc.max_rel);
    // one ballot per field: only fields nonzero somewhere in the warp are reduced
    const unsigned b0 = __ballot_sync(FULL, acc.dbytes != 0), b1 = __ballot_sync(FULL, acc.delems != 0);
    const unsigned b2 = __ballot_sync(FULL, acc.nan_r != 0), b3 = __ballot_sync(FULL, acc.nan_a != 0);
    const unsigned b4 = __ballot_sync(FULL, acc.nan_pos != 0), b5 = __ballot_sync(FULL, acc.rel_undef != 0);
    const unsigned b6 = __ballot_sync(FULL, acc.fail != 0), b7 = __ballot_sync(FULL, acc.max_ulp != 0);
    const unsigned b8 = __ballot_sync(FULL, mabs != 0), b9 = __ballot_sync(FULL, mrel != 0);
    if (b0 | b1 | b2 | b3 | b4 | b5 | b6 | b7 | b8 | b9) {
        const unsigned long long s0 = b0 ? warp_sum(acc.dbytes) : 0, s1 = b1 ? warp_sum(acc.delems) : 0,
                                 s2 = b2 ? warp_sum(acc.nan_r) : 0, s3 = b3 ? warp_sum(acc.nan_a) : 0,
                                 s4 = b4 ? warp_sum(acc.nan_pos) : 0, s5 = b5 ? warp_sum(acc.rel_undef) : 0,
                                 s6 = b6 ? warp_sum(acc.fail) : 0;
        const unsigned long long m0 = b7 ? warp_maxu(acc.max_ulp) : 0, m1 = b8 ? warp_maxu(mabs) : 0,
                                 m2 = b9 ? warp_maxu(mrel) : 0;
        if (lane == 0) {
            if (s0) atomicAdd((unsigned long long*)&rep->differing_bytes, s0);
            if (s1) atomicAdd((unsigned long long*)&rep->differing_elems, s1);
            if (s2) atomicAdd((unsigned long long*)&rep->nan_ref, s2);
            if (s3) atomicAdd((unsigned long long*)&rep->nan_act, s3);
            if (s4) atomicAdd((unsigned long long*)&rep->nan_pos_mismatch, s4);
            if (s5) atomicAdd((unsigned long long*)&rep->rel_undefined, s5);
            if (s6) atomicAdd((unsigned long long*)&rep->allclose_fail, s6);
            if (m0) atomicMax((unsigned long long*)&rep->max_ulp, m0);
            // non-negative doubles order like their bit patterns (+0.0 < ... < +inf)
            if (m1) atomicMax((unsigned long long*)&rep->max_abs, m1);
            if (m2) atomicMax((unsigned long long*)&rep->max_rel, m2);
        }
    }
    const uint32_t any = acc.any;
    acc_zero(acc);
    acc.any = any;
}

// One launch per dtype group: segments [seg0, seg0+nseg) own the global units
// [unit0, unit0+U).
// Unit order.  Segments of >= 4 MiB on average (and filtered launches): units
// are interleaved over warps (u = unit0 + w + k*W), so work that clusters (one
// planted buffer among identical ones, the dirty chunks of a filtered launch)
// spreads evenly; one contiguous block per warp left c3's Q/K/V warps idle
// while the O warps ran the element path (3.56 vs 5.27 TB/s), and the
// interleaved order also streams large pairs faster.  Smaller segments: one
// contiguous block per warp, walked segment by segment (interleaving made
// every unit a segment change, 1 MiB x 10k pairs 7.0 -> 6.2 TB/s).
// KC_K2_BLOCKED=0/1 forces either (measurement knob).  Filtered (K5 ran
// first): a unit whose chunk is clean is skipped without reading it.
template <int DT, int U, int Q2>
__device__ __forceinline__ void q_fin(typename QT_<DT>::T* q, uint32_t& qn, uint32_t* rq, uint32_t& rn, Acc& acc,
                                      double atol, double rtol, int equal_nan, int lane) {
    if constexpr (DT_<DT>::F && DT_<DT>::S == 2 && Q2 && !kGenericScan16)
        q_finish16<DT>(q, qn, rq, rn, acc, atol, rtol, equal_nan, lane);
    else
        q_finish<DT>(q, qn, acc, atol, rtol, equal_nan, lane);
}

template <int DT, int THREADS, int MINB, int VU, int Q2>
__global__ void __launch_bounds__(THREADS, MINB)
    k2_diff(const SegDev* __restrict__ segs, int seg0, int nseg, uint64_t unit0, uint64_t U,
            kc_diff_report* __restrict__ reps, unsigned long long* __restrict__ bitmaps, double atol, double rtol,
            int equal_nan, const unsigned long long* __restrict__ filter, int blocked, uint32_t flush_units) {
    const int lane = threadIdx.x & 31;
    segs += seg0;
    const uint64_t W = (uint64_t)gridDim.x * (THREADS / 32);
    const uint64_t w = (uint64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
    // blocks of B units, block b to warp b mod W: single units (interleaved)
    // when filtered or when segments are large; one contiguous block per warp
    // when the host chose `blocked` (small segments: a warp walks them in order)
    const uint64_t B = (filter || !blocked) ? 1 : (U + W - 1) / W;
    const uint64_t nblk = (U + B - 1) / B;
    if (w >= nblk) return;
    const uint64_t u0 = unit0 + w * B;
    int s = 0;
    {
        int lo = 0, hi = nseg;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (segs[mid].unit_off <= u0) lo = mid + 1; else hi = mid;
        }
        s = lo - 1;
    }
    Acc acc;
    acc_zero(acc);
    acc.alo = __double2float_rd(atol);
    acc.ahi = __double2float_ru(atol);
    acc.rlo = __double2float_rd(rtol);
    acc.rhi = __double2float_ru(rtol);
    extern __shared__ __align__(16) uint8_t k2_smem[];
    typename QT_<DT>::T* q =
        reinterpret_cast<typename QT_<DT>::T*>(k2_smem + (size_t)(threadIdx.x >> 5) * KQ<DT, VU>::kBytes);
    uint32_t qn = 0;  // warp-uniform queue length
    uint32_t* rq = reinterpret_cast<uint32_t*>(k2_smem + (size_t)(THREADS / 32) * KQ<DT, VU>::kBytes +
                                               (size_t)(threadIdx.x >> 5) * kRareBytes);
    uint32_t rn = 0;  // warp-uniform rare-queue length (16-bit floats, Q2)
    uint64_t since_flush = 0;
    for (uint64_t b = w; b < nblk; b += W)
    for (uint64_t u = unit0 + b * B, ue = min(unit0 + (b + 1) * B, unit0 + U); u < ue; ++u) {
        if (s + 1 < nseg && segs[s + 1].unit_off <= u) {
            // leaving segment s: flush what this warp accumulated for it, then
            // jump (binary search) to u's segment -- with units W apart a warp
            // can pass thousands of small segments it never touches
            q_fin<DT, VU, Q2>(q, qn, rq, rn, acc, atol, rtol, equal_nan, lane);
            acc_flush(acc, reps + segs[s].report, lane);
            ++s;  // contiguous blocks: the next segment
            if (s + 1 < nseg && segs[s + 1].unit_off <= u) {
                int lo = s + 1, hi = nseg;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (segs[mid].unit_off <= u) lo = mid + 1; else hi = mid;
                }
                s = lo - 1;
            }
        }
        const SegDev sg = segs[s];
        const uint32_t s_rep = sg.report;
        const uint64_t off = (u - sg.unit_off) * (uint64_t)kDiffUnit;
        if (filter) {
            const uint64_t c = sg.filter_chunk0 + off / kChunk;
            if (!((__ldg(filter + (c >> 6)) >> (c & 63)) & 1ULL)) continue;  // clean chunk
        }
        const uint32_t len = (uint32_t)min((uint64_t)kDiffUnit, sg.nbytes - off);
        const uint8_t* R = reinterpret_cast<const uint8_t*>(sg.ref) + off;
        const uint8_t* A = reinterpret_cast<const uint8_t*>(sg.act) + off;
        const bool vec_ok = ((sg.ref | sg.act) & 31) == 0;
        acc.any = 0;
        diff_unit<DT, VU, Q2>(R, A, len, vec_ok, acc, atol, rtol, equal_nan, lane, q, qn, rq, rn);
        if (__any_sync(0xFFFFFFFFu, acc.any) && lane == 0 && bitmaps) {
            const uint64_t k = sg.bitmap_chunk0 + off / kChunk;
            atomicOr(bitmaps + sg.bitmap_word0 + k / 64, 1ULL << (k % 64));
        }
        if (++since_flush == flush_units) {  // keeps the 32-bit lane counters in range
            since_flush = 0;
            q_fin<DT, VU, Q2>(q, qn, rq, rn, acc, atol, rtol, equal_nan, lane);
            acc_flush(acc, reps + s_rep, lane);
        }
    }
    q_fin<DT, VU, Q2>(q, qn, rq, rn, acc, atol, rtol, equal_nan, lane);
    acc_flush(acc, reps + segs[s].report, lane);
}

// per report: nbytes / n_elems / n_chunks / percent / pass
__global__ void k2_finalize(const ReportMeta* __restrict__ meta, int nrep, kc_diff_report* __restrict__ reps) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nrep) return;
    kc_diff_report& r = reps[j];
    const int dt = meta[j].dtype;
    const int es = (dt == KC_DT_BYTES || dt == KC_DT_U8 || dt == KC_DT_I8) ? 1
                   : (dt == KC_DT_U16 || dt == KC_DT_I16 || dt == KC_DT_F16 || dt == KC_DT_BF16) ? 2
                   : (dt == KC_DT_U32 || dt == KC_DT_I32 || dt == KC_DT_F32) ? 4 : 8;
    const uint64_t n = meta[j].nbytes;
    r.nbytes = n;
    r.n_elems = n / es;
    r.n_chunks = (n + kChunk - 1) / kChunk;
    r.percent_bytes = n ? __ddiv_rn(__dmul_rn(100.0, (double)r.differing_bytes), (double)n) : 0.0;
    if (dt == KC_DT_BYTES) {
        r.differing_elems = r.differing_bytes;
        r.pass = r.differing_bytes == 0;
    } else if (dt == KC_DT_F16 || dt == KC_DT_BF16 || dt == KC_DT_F32 || dt == KC_DT_F64) {
        r.pass = r.allclose_fail == 0;
    } else {
        r.pass = r.differing_elems == 0;
    }
}

// ========================================================================== //
// K4: gather/scatter of many small ranges (pack small regions for one DMA).  //
// ========================================================================== //
__global__ void k4_gather(const uint64_t* __restrict__ src, const uint64_t* __restrict__ dst,
                          const uint64_t* __restrict__ len, int n) {
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const uint8_t* s = reinterpret_cast<const uint8_t*>(src[i]);
        uint8_t* d = reinterpret_cast<uint8_t*>(dst[i]);
        const uint64_t L = len[i];
        if (((src[i] | dst[i]) & 15) == 0) {
            const uint64_t nv = L / 16;
            for (uint64_t k = threadIdx.x; k < nv; k += blockDim.x)
                reinterpret_cast<uint4*>(d)[k] = __ldg(reinterpret_cast<const uint4*>(s) + k);
            for (uint64_t k = nv * 16 + threadIdx.x; k < L; k += blockDim.x) d[k] = s[k];
        } else {
            for (uint64_t k = threadIdx.x; k < L; k += blockDim.x) d[k] = s[k];
        }
    }
}

// ========================================================================== //
// launchers                                                                  //
// ========================================================================== //
using TmaA = HkCfg<256, 3, 1024>;  // 64 slots x 3 x 1 KiB
using TmaB = HkCfg<128, 3, 2048>;  // 32 slots x 3 x 2 KiB
using CpA = CpCfg<8, 3, 1024>;   // 64 chunks/SM x 3 x 1 KiB   (default: HBM-bound)
using CpA0 = CpCfg<8, 3, 1024, false>;  // round 2's padded (unswizzled) slices, for A/B
using CpD = CpCfg<16, 3, 512>;   // 128 chunks/SM x 3 x 512 B
using CpS = CpCfg<2, 6, 1024>;   // small snapshots: 2-warp CTAs, 6-deep rings, so < 148 x 64 chunks still
                                 // spread over every SM (a chunk's hash is a ~25 us serial chain)
using Ws1 = WsCfg<1, 4, 2048>;  // one CTA per SM, HW hashing warps (one per SMSP) + HW producers
using Ws2 = WsCfg<2, 4, 2048>;  // on SMSP 3, 4 x 2 KiB slices (64 rounds between ring hand-overs)
using Ws3 = WsCfg<3, 4, 2048>;
using CmpA = CmpCfg<8, 3, 512>;  // K5: 64 chunk pairs/SM x 3 x (512 B act + 512 B ref)

cudaError_t kernels_init() {
    cudaError_t e = cudaFuncSetAttribute(k1_hash_tma<TmaA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmaA::kSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k1_hash_tma<TmaB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TmaB::kSmem);
#define KC_CP_ATTR(CFG)                                                                                      \
    if (e == cudaSuccess)                                                                                    \
        e = cudaFuncSetAttribute(k1_hash_cpasync<CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CFG::kSmem);
    KC_CP_ATTR(CpA) KC_CP_ATTR(CpD) KC_CP_ATTR(CpS) KC_CP_ATTR(CpA0)
#undef KC_CP_ATTR
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k1_hash_cpasync<CpA, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)CpA::kSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k1_hash_cpasync<CpS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)CpS::kSmem);
#define KC_WS_ATTR(CFG)                                                                                      \
    if (e == cudaSuccess)                                                                                    \
        e = cudaFuncSetAttribute(k1_hash_ws<CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CFG::kSmem);
    KC_WS_ATTR(Ws1) KC_WS_ATTR(Ws2) KC_WS_ATTR(Ws3)
#undef KC_WS_ATTR
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k5_hash_cmp<CmpA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CmpA::kSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k5_hash_cmp<CmpA, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)CmpA::kSmem);
    return e;
}

// Grid for the group-interleaved ring kernels (K1/K5/K6): warp w hashes groups
// j0, j0 + W, ... (W = warps in the grid).  With groups = 3.5 x the warps that
// fit, half the warps would run a 4th group alone, a latency-bound tail (2 GiB
// went at 6.0 TB/s).  With few groups per warp the grid shrinks until every
// warp gets the same count (6.3 TB/s); large snapshots keep the full grid.
static uint64_t balanced_grid(uint64_t groups, uint64_t max_ctas, int warps_per_cta) {
    const uint64_t max_warps = max_ctas * (uint64_t)warps_per_cta;
    uint64_t warps = std::min(groups, max_warps);
    const uint64_t per_warp = (groups + max_warps - 1) / max_warps;
    if (per_warp > 1 && per_warp <= 16) warps = (groups + per_warp - 1) / per_warp;
    return (warps + warps_per_cta - 1) / warps_per_cta;
}

cudaError_t launch_hash_cmp(const PairDev* d_pairs, int npair, uint64_t C, uint64_t* d_out, uint64_t* d_dirty,
                            const uint32_t* map, int num_sms, cudaStream_t s, bool self) {
    if (C == 0) return cudaSuccess;
    const uint64_t groups = (C + 7) / 8;
    const uint64_t grid = balanced_grid(groups, (uint64_t)num_sms, CmpA::kWarps);
    if (self)
        k5_hash_cmp<CmpA, true><<<(unsigned)grid, CmpA::kWarps * 32, CmpA::kSmem, s>>>(
            d_pairs, npair, C, d_out, reinterpret_cast<unsigned long long*>(d_dirty), map);
    else
        k5_hash_cmp<CmpA><<<(unsigned)grid, CmpA::kWarps * 32, CmpA::kSmem, s>>>(
            d_pairs, npair, C, d_out, reinterpret_cast<unsigned long long*>(d_dirty), map);
    return cudaGetLastError();
}

template <class CFG>
static void launch_tma(const RegionDev* d_regs, int nreg, uint64_t C, uint64_t* d_out, const uint32_t* map,
                       int num_sms, cudaStream_t s) {
    uint64_t grid = (C + CFG::kSlots - 1) / CFG::kSlots;
    if (grid > (uint64_t)num_sms) grid = num_sms;
    k1_hash_tma<CFG><<<(unsigned)grid, CFG::kThreads, CFG::kSmem, s>>>(d_regs, nreg, C, d_out, map);
}

template <class CFG>
static void launch_cp(const RegionDev* d_regs, int nreg, uint64_t C, uint64_t* d_out, const uint32_t* map,
                      int num_sms, cudaStream_t s, const unsigned long long* d_dst = nullptr,
                      const uint32_t* order = nullptr) {
    const uint64_t groups = (C + 7) / 8;
    // at most 8 warps' worth of CTAs per SM (one CTA of the 8-warp configs, four of CpS)
    const uint64_t per_sm = std::min<uint64_t>(CFG::kWarps >= 8 ? 1 : 8 / CFG::kWarps,
                                               std::max<uint64_t>(1, 232448 / (CFG::kSmem + 1024)));  // + smem fit
    const uint64_t grid = balanced_grid(groups, (uint64_t)num_sms * per_sm, CFG::kWarps);
    if (d_dst)
        k1_hash_cpasync<CFG, true><<<(unsigned)grid, CFG::kWarps * 32, CFG::kSmem, s>>>(d_regs, nreg, C, d_out, map,
                                                                                       d_dst, order);
    else
        k1_hash_cpasync<CFG><<<(unsigned)grid, CFG::kWarps * 32, CFG::kSmem, s>>>(d_regs, nreg, C, d_out, map,
                                                                                 nullptr, order);
}

// Sub-wave K1 with one hashing warp alone on each SMSP: a second chain-bound warp on the same
// SMSP shares its FMA pipe (~17 pipe cycles per round each) and stretches the ~30-cycle round
// to 45-50 (tools/probes/k1_round_probe.cu at 256 threads/CTA).  One CTA per SM with HW =
// ceil(groups / SMs) <= 3 hashing warps on SMSPs 0..HW-1 and their producers on SMSP 3.  With
// HW = 4 the producers must share SMSPs with hashing warps, and CpS (2-warp CTAs staging their
// own rings, one warp per SMSP at that size) measured faster (1 MiB x 256: 49.2 vs 52.2 us).
template <class W1, class W2, class W3>
static bool launch_ws_subwave(const RegionDev* d_regs, int nreg, uint64_t C, uint64_t* d_out, const uint32_t* map,
                              int num_sms, cudaStream_t s, const uint32_t* order) {
    const uint64_t groups = (C + 7) / 8;
    const uint64_t hw = (groups + num_sms - 1) / num_sms;
    if (hw > 3) return false;
    const unsigned grid = (unsigned)((groups + hw - 1) / hw);
    switch (hw) {
        case 1: k1_hash_ws<W1><<<grid, W1::kWarps * 32, W1::kSmem, s>>>(d_regs, nreg, C, d_out, map, order); break;
        case 2: k1_hash_ws<W2><<<grid, W2::kWarps * 32, W2::kSmem, s>>>(d_regs, nreg, C, d_out, map, order); break;
        default: k1_hash_ws<W3><<<grid, W3::kWarps * 32, W3::kSmem, s>>>(d_regs, nreg, C, d_out, map, order); break;
    }
    return true;
}

// K1 variant selection (KC_K1_VARIANT, tuning knob; default = the measured best)
static int k1_variant() {
    static int v = [] {
        const char* e = getenv("KC_K1_VARIANT");
        return e && *e ? atoi(e) : 0;
    }();
    return v;
}

cudaError_t launch_hash(const RegionDev* d_regs, int nreg, uint64_t C, bool aligned, uint64_t* d_out,
                        const uint32_t* map, int num_sms, cudaStream_t s, const uint32_t* order) {
    if (C == 0) return cudaSuccess;
    if (!aligned) {
        uint64_t grid = (C + 63) / 64;
        if (grid > (uint64_t)num_sms * 8) grid = num_sms * 8;
        k1_hash_generic<<<(unsigned)grid, 256, 0, s>>>(d_regs, nreg, C, d_out, map);
        return cudaGetLastError();
    }
    // measured on B200: cp.async 64 chunks x 3 x 1 KiB is HBM-bound
    switch (k1_variant()) {
        case 1: launch_tma<TmaA>(d_regs, nreg, C, d_out, map, num_sms, s); break;
        case 2: launch_tma<TmaB>(d_regs, nreg, C, d_out, map, num_sms, s); break;
        case 3: launch_cp<CpD>(d_regs, nreg, C, d_out, map, num_sms, s, nullptr, order); break;
        case 9: launch_cp<CpA0>(d_regs, nreg, C, d_out, map, num_sms, s, nullptr, order); break;
        case 4:  // round 2's sub-wave path (CpS below one wave), for A/B
            if ((C + 7) / 8 < (uint64_t)num_sms * 8)
                launch_cp<CpS>(d_regs, nreg, C, d_out, map, num_sms, s, nullptr, order);
            else
                launch_cp<CpA>(d_regs, nreg, C, d_out, map, num_sms, s, nullptr, order);
            break;
        default:
            // up to 3 x SMs groups: one hashing warp per SMSP fed by producer warps (c2 45.3 ->
            // 38.7 us back to back, 64 KiB x 1k 48.0 -> 38.9 us; K1); then, below one
            // wave of 8-warp CTAs, CpS spread over every SM (round 2 A/B on c2: a per-quad TMA
            // bulk ring of 16 slots x 3 x 2 KiB 92-129 us; a warp ring filled by one bulk copy per
            // chunk slice from the quad leaders, 66 us; CpS 48-50 us); above, CpA
            if (launch_ws_subwave<Ws1, Ws2, Ws3>(d_regs, nreg, C, d_out, map, num_sms, s, order)) break;
            if ((C + 7) / 8 < (uint64_t)num_sms * 8)
                launch_cp<CpS>(d_regs, nreg, C, d_out, map, num_sms, s, nullptr, order);
            else
                launch_cp<CpA>(d_regs, nreg, C, d_out, map, num_sms, s, nullptr, order);
            break;
    }
    return cudaGetLastError();
}

cudaError_t launch_hash_copy(const RegionDev* d_regs, int nreg, uint64_t C, uint64_t* d_out,
                             const unsigned long long* d_dst, const uint32_t* map, int num_sms, cudaStream_t s,
                             const uint32_t* order) {
    if (C == 0) return cudaSuccess;
    if ((C + 7) / 8 < (uint64_t)num_sms * 8)
        launch_cp<CpS>(d_regs, nreg, C, d_out, map, num_sms, s, d_dst, order);
    else
        launch_cp<CpA>(d_regs, nreg, C, d_out, map, num_sms, s, d_dst, order);
    return cudaGetLastError();
}

cudaError_t launch_digests(const RegionDev* d_regs, int nreg, const uint64_t* d_h, uint64_t* d_dig, uint8_t* d_scratch,
                           uint64_t* d_snap, cudaStream_t s) {
    if (nreg == 0) return cudaSuccess;
    const int grid = std::min(nreg, 148 * 8);
    k1_region_digest<<<grid, 32, 0, s>>>(d_regs, nreg, d_h, d_dig, d_snap ? d_scratch : nullptr);
    if (d_snap) k1_snapshot_digest<<<1, 4, 0, s>>>(d_scratch, nreg, d_snap);
    return cudaGetLastError();
}

cudaError_t launch_snapshot_digest(const uint8_t* d_triples, int nreg, uint64_t* d_out, cudaStream_t s) {
    k1_snapshot_digest<<<1, 4, 0, s>>>(d_triples, nreg, d_out);
    return cudaGetLastError();
}

cudaError_t launch_written(const uint64_t* d_pre, const uint64_t* d_post, uint64_t C, uint64_t* d_bitmap,
                           uint64_t* d_count, int num_sms, cudaStream_t s) {
    if (C == 0) return cudaSuccess;
    const uint64_t nwords = (C + 63) / 64;
    uint64_t grid = (nwords + 7) / 8;
    if (grid > (uint64_t)num_sms * 4) grid = num_sms * 4;
    k3_written<<<(unsigned)grid, 256, 0, s>>>(d_pre, d_post, C, d_bitmap, (unsigned long long*)d_count);
    return cudaGetLastError();
}

// K2 launch configurations (KC_K2_VARIANT, tuning knob): threads per CTA,
// min CTAs per SM (register budget), vectors of each operand in flight per lane
// contiguous unit blocks for groups of small segments (see k2_diff)
static int k2_blocked(const DiffGroup& G) {
    static const int forced = [] {
        const char* e = getenv("KC_K2_BLOCKED");
        return e && *e ? atoi(e) : -1;
    }();
    if (forced >= 0) return forced;
    return G.n_units < 256 * (uint64_t)G.n_segs;  // average segment < 4 MiB
}

template <int DT, int THREADS, int MINB, int U, int Q2 = 1>
static void launch_k2_cfg(const SegDev* d_segs, const DiffGroup& G, kc_diff_report* d_reps,
                          unsigned long long* bm, double atol, double rtol, int equal_nan, int num_sms,
                          cudaStream_t s, const unsigned long long* filter) {
    constexpr int WPB = THREADS / 32;
    uint64_t grid = (G.n_units + WPB - 1) / WPB;
    if (grid > (uint64_t)num_sms * MINB) grid = (uint64_t)num_sms * MINB;
    // KC_K2_MAX_CTAS (tests only): fewer CTAs, so each warp walks many units and
    // segment boundaries (with KC_K2_FLUSH_UNITS: many periodic flushes)
    static const uint64_t max_ctas = [] {
        const char* e = getenv("KC_K2_MAX_CTAS");
        const long v = e && *e ? strtol(e, nullptr, 10) : 0;
        return v > 0 ? (uint64_t)v : ~0ull;
    }();
    if (grid > max_ctas) grid = max_ctas;
    constexpr int smem = DT_<DT>::F ? WPB * (KQ<DT, U>::kBytes + (DT_<DT>::S == 2 ? kRareBytes : 0)) : 0;
    static bool attr = [] {
        return cudaFuncSetAttribute(k2_diff<DT, THREADS, MINB, U, Q2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem) == cudaSuccess;
    }();
    (void)attr;
    // KC_K2_FLUSH_UNITS (tests only): flush the lane accumulators every n units
    // instead of every kFlushUnits (1 GiB per warp, which no test-sized launch
    // reaches), so the periodic-flush path is exercised
    static const uint32_t flush_units = [] {
        const char* e = getenv("KC_K2_FLUSH_UNITS");
        const long v = e && *e ? strtol(e, nullptr, 10) : 0;
        return v > 0 && v <= (long)kFlushUnits ? (uint32_t)v : (uint32_t)kFlushUnits;
    }();
    k2_diff<DT, THREADS, MINB, U, Q2><<<(unsigned)grid, THREADS, smem, s>>>(d_segs, G.seg0, G.n_segs, G.unit0, G.n_units,
                                                                         d_reps, bm, atol, rtol, equal_nan, filter,
                                                                         k2_blocked(G), flush_units);
}

// Measured on B200 (tools/k2_bench.py): 512 threads x 1 CTA per
// SM with 2 vectors of each operand in flight keeps the float paths free of
// spills and reaches 6.9 TB/s on identical bf16 pairs; 512 x 2 CTAs (64
// registers) spilled segment state into the inner loop (3.6 TB/s).  For the
// planted 16-bit case 640 / 768 threads (1 or 2 vectors) were no faster
// (profiles/r1_k2_bench_fast16_configs.txt).
template <int DT>
static void launch_k2(const SegDev* d_segs, const DiffGroup& G, kc_diff_report* d_reps, unsigned long long* bm,
                      double atol, double rtol, int equal_nan, int num_sms, cudaStream_t s,
                      const unsigned long long* filter) {
    if constexpr (DT_<DT>::F && DT_<DT>::S == 2) {
        // KC_K2_Q2 (A/B measurement knob; profiles/r2_k2_bench.txt): 0 = the round-1
        // 16-bit element path, 1 = the rare queue with the integer flag scan,
        // 2 = + the HSET2 flag scan (vec_scan16h), 3 (default) = + LEA.HI pushes
        static const int q2 = [] {
            const char* e = getenv("KC_K2_Q2");
            return e && *e ? atoi(e) : 3;
        }();
        if (q2 == 0) {
            launch_k2_cfg<DT, 512, 1, 2, 0>(d_segs, G, d_reps, bm, atol, rtol, equal_nan, num_sms, s, filter);
            return;
        }
        if (q2 == 2) {
            launch_k2_cfg<DT, 512, 1, 2, 2>(d_segs, G, d_reps, bm, atol, rtol, equal_nan, num_sms, s, filter);
            return;
        }
        if (q2 == 3) {
            launch_k2_cfg<DT, 512, 1, 2, 3>(d_segs, G, d_reps, bm, atol, rtol, equal_nan, num_sms, s, filter);
            return;
        }
    }
    if constexpr (!DT_<DT>::F) {
        // sub-wave launches (at most ~4 units per warp of the full grid) are bound by
        // load round trips, not bandwidth: 4 vectors of each operand in flight per lane
        // instead of 2 halves the trips per unit (integer and byte dtypes: no element
        // queue, so the registers are there)
        static const bool small_u4 = [] {
            const char* e = getenv("KC_K2_SMALL_U4");
            return !(e && *e == '0');
        }();
        // (likewise many short segments: a warp walks them one by one, a few round
        // trips each, when at least half the segments are a single 16 KiB unit)
        if (small_u4 && !filter &&
            (G.n_units <= (uint64_t)num_sms * 16 * 4 || 2 * (uint64_t)G.n_segs >= G.n_units)) {
            launch_k2_cfg<DT, 512, 1, 4, 1>(d_segs, G, d_reps, bm, atol, rtol, equal_nan, num_sms, s, filter);
            return;
        }
    }
    launch_k2_cfg<DT, 512, 1, 2, 1>(d_segs, G, d_reps, bm, atol, rtol, equal_nan, num_sms, s, filter);
}

cudaError_t launch_diff(const SegDev* d_segs, const DiffGroup* groups, int ngroups, const ReportMeta* d_meta,
                        int nrep, kc_diff_report* d_reps, uint64_t* d_bitmaps, double atol, double rtol,
                        int equal_nan, int num_sms, cudaStream_t s, const uint64_t* d_filter) {
    const unsigned long long* filter = reinterpret_cast<const unsigned long long*>(d_filter);
    for (int g = 0; g < ngroups; ++g) {
        const DiffGroup& G = groups[g];
        if (G.n_units == 0 || G.n_segs == 0) continue;
        unsigned long long* bm = (unsigned long long*)d_bitmaps;
        switch (G.dtype) {
#define KC_CASE(D) \
    case D: launch_k2<D>(d_segs, G, d_reps, bm, atol, rtol, equal_nan, num_sms, s, filter); break;
            KC_CASE(KC_DT_BYTES) KC_CASE(KC_DT_U8) KC_CASE(KC_DT_I8) KC_CASE(KC_DT_U16) KC_CASE(KC_DT_I16)
            KC_CASE(KC_DT_U32) KC_CASE(KC_DT_I32) KC_CASE(KC_DT_U64) KC_CASE(KC_DT_I64) KC_CASE(KC_DT_F16)
            KC_CASE(KC_DT_BF16) KC_CASE(KC_DT_F32) KC_CASE(KC_DT_F64)
#undef KC_CASE
            default: return cudaErrorInvalidValue;
        }
    }
    if (nrep > 0) k2_finalize<<<(nrep + 127) / 128, 128, 0, s>>>(d_meta, nrep, d_reps);
    return cudaGetLastError();
}

cudaError_t launch_gather(const uint64_t* d_src, const uint64_t* d_dst, const uint64_t* d_len, int n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k4_gather<<<min(n, 148 * 8), 256, 0, s>>>(d_src, d_dst, d_len, n);
    return cudaGetLastError();
}

}  // namespace kc
