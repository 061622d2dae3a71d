// kc_attn_fwd.cu -- F4 workload: an attention-forward
// kernel in the shape of the Triton tutorial attn_fwd the paper measures
// (fp16, B=2, H=16, S=4096, D=128), compiled once per
// "autotune config" KC_ATTN_BLOCK_N into synth/kc_attn_fwd_n<BN>.cubin.  All
// configs export the same symbol, like the configs of one @triton.autotune
// kernel, so a captured dispatch of one config can be replayed with another
// config's code object (kc_replay image_override) and validated with K2.
//
// It is workload, not the hot path: plain CUDA-core fp32 arithmetic, fixed
// accumulation order within a config, so every config is bit-reproducible and
// two configs differ only where BLOCK_N moves the online-softmax rescale points
// (the paper's attribution: "the BLOCK_N tile ... reorders the
// softmax-denominator reduction across the K dimension").
//
// Per key block of BLOCK_N (Triton _attn_fwd_inner order):
//   qk    = q . k^T                       (fp32, d = 0..127 in order)
//   m_ij  = max(m_i, rowmax(qk) * qk_scale),   qk_scale = sm_scale * log2(e)
//   p     = exp2(qk * qk_scale - m_ij)
//   l_ij  = rowsum(p);  alpha = exp2(m_i - m_ij);  l_i = l_i * alpha + l_ij
//   acc   = acc * alpha;  acc += fp16(p) . v     (fp32, keys in order)
//   m_i   = m_ij
// out = fp16(acc / l_i).
//
// Layout: Q, K, V, O contiguous [B][H][S][128] fp16; grid (S/BLOCK_M, B*H),
// block 4*BLOCK_M: BLOCK_M = 64 query rows per CTA by default, 4 threads per row.  Thread (r, c4):
// score columns n = c4 + 4j of each 32-key sub-tile, output columns
// c4*32 .. c4*32+31.  Requires S % BLOCK_N == 0 and S % 64 == 0.
#include <cuda_fp16.h>
#include <stdint.h>

#ifndef KC_ATTN_BLOCK_N
#define KC_ATTN_BLOCK_N 64
#endif
#ifndef KC_ATTN_BLOCK_M  // query rows per CTA (4 threads each); does not change any row's arithmetic
#define KC_ATTN_BLOCK_M 64
#endif

namespace {
constexpr int D = 128, BM = KC_ATTN_BLOCK_M, SUB = 32, PAD = 8, T = 4 * BM;
constexpr int BN = KC_ATTN_BLOCK_N;
static_assert(BN % SUB == 0, "BLOCK_N must be a multiple of 32");
constexpr int NSUB = BN / SUB;
constexpr int QS = D + PAD;   // smem row pitch (halves) of the Q and K/V tiles
constexpr int PS = BN + PAD;  // smem row pitch (halves) of P

__device__ __forceinline__ void load_tile(__half* dst, const __half* src, int rows, int tid) {
    // rows x 128 halves, 16-byte vectors, T threads
    for (int v = tid; v < rows * (D / 8); v += T) {
        const int r = v / (D / 8), c = (v % (D / 8)) * 8;
        *reinterpret_cast<uint4*>(dst + r * QS + c) = *reinterpret_cast<const uint4*>(src + (size_t)r * D + c);
    }
}

__device__ __forceinline__ void h8_to_f(const __half* p, float* f) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __half22float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
}  // namespace

extern "C" __global__ void __launch_bounds__(4 * KC_ATTN_BLOCK_M) kc_fixture_attn_fwd(const __half* __restrict__ Q,
                                                                      const __half* __restrict__ K,
                                                                      const __half* __restrict__ V,
                                                                      __half* __restrict__ O, int S, float sm_scale) {
    __shared__ __align__(16) __half qs[BM * QS];
    __shared__ __align__(16) __half kv[SUB * QS];
    __shared__ __align__(16) __half ps[BM * PS];
    const int tid = threadIdx.x, r = tid >> 2, c4 = tid & 3;
    const size_t head = (size_t)blockIdx.y * S * D;
    const int m0 = blockIdx.x * BM;
    const float qk_scale = sm_scale * 1.44269504f;
    load_tile(qs, Q + head + (size_t)m0 * D, BM, tid);

    float m_i = -INFINITY, l_i = 0.f;
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;

    for (int n0 = 0; n0 < S; n0 += BN) {
        // ---- qk = q . k^T over the BLOCK_N keys, in 32-key sub-tiles
        float s[NSUB * 8];
#pragma unroll
        for (int i = 0; i < NSUB * 8; ++i) s[i] = 0.f;
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb) {
            __syncthreads();
            load_tile(kv, K + head + (size_t)(n0 + sb * SUB) * D, SUB, tid);
            __syncthreads();
            for (int d0 = 0; d0 < D; d0 += 8) {
                float q8[8];
                h8_to_f(qs + r * QS + d0, q8);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float k8[8];
                    h8_to_f(kv + (c4 + 4 * j) * QS + d0, k8);
                    float a = s[sb * 8 + j];
#pragma unroll
                    for (int e = 0; e < 8; ++e) a = fmaf(q8[e], k8[e], a);
                    s[sb * 8 + j] = a;
                }
            }
        }
        // ---- online softmax (row = 4 consecutive lanes; fixed shuffle order)
        float mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < NSUB * 8; ++i) mx = fmaxf(mx, s[i]);
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, 2));
        const float m_ij = fmaxf(m_i, mx * qk_scale);
        float l_ij = 0.f;
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float p = exp2f(s[sb * 8 + j] * qk_scale - m_ij);
                l_ij += p;
                ps[r * PS + sb * SUB + c4 + 4 * j] = __float2half_rn(p);
            }
        l_ij += __shfl_xor_sync(0xFFFFFFFFu, l_ij, 1);
        l_ij += __shfl_xor_sync(0xFFFFFFFFu, l_ij, 2);
        const float alpha = exp2f(m_i - m_ij);
        l_i = l_i * alpha + l_ij;
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] *= alpha;
        m_i = m_ij;
        // ---- acc += fp16(p) . v, keys in order
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb) {
            __syncthreads();  // also publishes ps before the first sub-tile
            load_tile(kv, V + head + (size_t)(n0 + sb * SUB) * D, SUB, tid);
            __syncthreads();
            for (int n = 0; n < SUB; ++n) {
                const float p = __half2float(ps[r * PS + sb * SUB + n]);
#pragma unroll
                for (int d0 = 0; d0 < 32; d0 += 8) {
                    float v8[8];
                    h8_to_f(kv + n * QS + c4 * 32 + d0, v8);
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[d0 + e] = fmaf(p, v8[e], acc[d0 + e]);
                }
            }
        }
    }
    // ---- epilogue: acc / l_i -> fp16, 64 contiguous bytes per thread
    __half* o = O + head + (size_t)(m0 + r) * D + c4 * 32;
#pragma unroll
    for (int d0 = 0; d0 < 32; d0 += 8) {
        __align__(16) __half h[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) h[e] = __float2half_rn(acc[d0 + e] / l_i);
        *reinterpret_cast<uint4*>(o + d0) = *reinterpret_cast<const uint4*>(h);
    }
}
