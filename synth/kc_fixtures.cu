// kc_fixtures.cu -- the synthetic "application" kernels whose dispatches are
// captured and replayed.  They are workload, not the hot
// path: compiled to synth/kc_fixtures.cubin and loaded through kc_capture's
// (image, mangled) dispatch description, exactly like a captured code object.
// Every kernel accumulates in a fixed order, so a replay is bit-reproducible.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

// KC_VARIANT_DELTA: a "modified kernel" for the validate-variant workflow
// (PAPER.md:1120-1126); 0 = the captured kernel.
#ifndef KC_VARIANT_DELTA
#define KC_VARIANT_DELTA 0
#endif

struct KcNode {
    unsigned long long next;  // device VA of the next node, 0 ends the list
    unsigned int value;
    unsigned int pad;
};

// F1 / F1': pointer-chasing linked-list walk (config c1).  Each thread walks
// one list from heads[i]; out[(va - nodes_base)/16] = running sum; mutate=1
// also rewrites value <- 3*value + 1 in place (the capture-mode probe; the
// KC_VARIANT_DELTA variant adds DELTA to both the sums and the rewrite).
extern "C" __global__ void kc_fixture_walk(const unsigned long long* __restrict__ heads, unsigned long long* out,
                                           unsigned long long nodes_base, unsigned int n_lists, int mutate) {
    const unsigned int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_lists) return;
    unsigned long long va = heads[i];
    unsigned long long acc = 0;
    while (va != 0) {
        KcNode* nd = reinterpret_cast<KcNode*>(va);
        const unsigned int v = nd->value;
        acc += v + KC_VARIANT_DELTA;
        out[(va - nodes_base) / 16] = acc;
        if (mutate) nd->value = v * 3u + 1u + KC_VARIANT_DELTA;
        va = nd->next;
    }
}

// F2: single-token decode attention over a fp16 KV cache (config c2, the
// llama.cpp-shaped snapshot).  q [H=32][D=64] fp16, k/v [L=4][KVH=8][CTX][64]
// fp16, GQA group 4, layer `layer`, first ctx_len positions valid.  One block
// of 128 threads per q head; scores, max, sum and the output accumulate in a
// fixed order (per-thread strided then a fixed shared-memory tree).
extern "C" __global__ void kc_fixture_decode_attn(const __half* __restrict__ q, const __half* __restrict__ kc,
                                                  const __half* __restrict__ vc, float* __restrict__ out,
                                                  float* __restrict__ scratch, int layer, int ctx, int ctx_len) {
    constexpr int D = 64, KVH = 8, H = 32, T = 128;
    const int h = blockIdx.x, tid = threadIdx.x, kvh = h / (H / KVH);
    const __half* K = kc + ((size_t)layer * KVH + kvh) * (size_t)ctx * D;
    const __half* V = vc + ((size_t)layer * KVH + kvh) * (size_t)ctx * D;
    float* S = scratch + (size_t)h * ctx;  // per-head score buffer (workspace region)
    __shared__ float red[T];
    __shared__ float qs[D];
    if (tid < D) qs[tid] = __half2float(q[h * D + tid]);
    __syncthreads();
    float m = -INFINITY;
    for (int t = tid; t < ctx_len; t += T) {
        float s = 0.f;
        for (int d = 0; d < D; ++d) s = fmaf(qs[d], __half2float(K[(size_t)t * D + d]), s);
        s *= 0.125f;  // 1/sqrt(64)
        S[t] = s;
        m = fmaxf(m, s);
    }
    red[tid] = m;
    __syncthreads();
    for (int o = T / 2; o > 0; o >>= 1) {
        if (tid < o) red[tid] = fmaxf(red[tid], red[tid + o]);
        __syncthreads();
    }
    m = red[0];
    __syncthreads();
    float l = 0.f;
    for (int t = tid; t < ctx_len; t += T) {
        const float p = __expf(S[t] - m);
        S[t] = p;
        l += p;
    }
    red[tid] = l;
    __syncthreads();
    for (int o = T / 2; o > 0; o >>= 1) {
        if (tid < o) red[tid] += red[tid + o];
        __syncthreads();
    }
    l = red[0];
    __syncthreads();
    // output: thread pair (d, half) accumulates over t in a fixed order
    const int d = tid & (D - 1), part = tid >> 6;
    float acc = 0.f;
    for (int t = part; t < ctx_len; t += 2) acc = fmaf(S[t], __half2float(V[(size_t)t * D + d]), acc);
    red[tid] = acc;
    __syncthreads();
    if (tid < D) out[h * D + tid] = (red[tid] + red[tid + D]) / l;
}

// F3: pointer-indirected MoE GEMV (config c4).  ptr_table holds 60 w13 expert
// pointers then 60 w2 expert pointers (device VAs inside the pool); for each
// token t and its top-2 experts, y[t][o] = sum_j sum_i W13[e_j][o][i] * x[t][i]
// (bf16 weights/activations, fp32 accumulation).  One warp per (t, o); lanes
// stride i, then a fixed xor-shuffle tree.
extern "C" __global__ void kc_fixture_moe_gemv(const unsigned long long* __restrict__ ptr_table,
                                               const __nv_bfloat16* __restrict__ x, const int* __restrict__ topk,
                                               float* __restrict__ y, int T, int O, int I) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= (long long)T * O) return;
    const int t = (int)(gw / O), o = (int)(gw % O);
    float acc = 0.f;
    for (int j = 0; j < 2; ++j) {
        const int e = topk[t * 2 + j];
        const __nv_bfloat16* W = reinterpret_cast<const __nv_bfloat16*>(ptr_table[e]) + (size_t)o * I;
        for (int i = lane; i < I; i += 32) acc = fmaf(__bfloat162float(W[i]), __bfloat162float(x[(size_t)t * I + i]), acc);
    }
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, s);
    if (lane == 0) y[(size_t)t * O + o] = acc;
}

// F3 (module variables): a kernel whose result depends on
// module state the tracker cannot see: a __constant__ table and a __device__
// scale the application sets after loading the module, plus a __device__
// counter the dispatch itself writes.
__constant__ unsigned int kc_fixture_cvals[8];
__device__ float kc_fixture_scale = 2.5f;
__device__ unsigned long long kc_fixture_hits;
extern "C" __global__ void kc_fixture_modvar(unsigned long long* out, unsigned int n) {
    const unsigned int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = (unsigned long long)((float)kc_fixture_cvals[i & 7] * kc_fixture_scale) + i;
    atomicAdd(&kc_fixture_hits, 1ull);
}

// F4 sequences: an elementwise step independent of the list walk,
// y[i] = a * x[i] + y[i] (u32, modulo 2^32: exact, so the oracle check is exact).
extern "C" __global__ void kc_fixture_axpy_u32(const unsigned int* __restrict__ x, unsigned int* __restrict__ y,
                                               unsigned int n, unsigned int a) {
    const unsigned int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = a * x[i] + y[i] + KC_VARIANT_DELTA;
}

// A dispatch with more than 48 KiB of dynamic shared memory (needs the opt-in
// function attribute on every module it is launched from): each block of 1024
// threads stages `per_block` u32 through shared memory and writes them reversed.
extern "C" __global__ void kc_fixture_smem_reverse(const unsigned int* __restrict__ in, unsigned int* __restrict__ out,
                                                   unsigned int per_block) {
    extern __shared__ unsigned int stage[];
    const size_t b0 = (size_t)blockIdx.x * per_block;
    for (unsigned int i = threadIdx.x; i < per_block; i += blockDim.x) stage[i] = in[b0 + i];
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < per_block; i += blockDim.x) out[b0 + i] = stage[per_block - 1 - i] ^ blockIdx.x;
}

// A dispatch launched with runtime thread-block clusters (cuLaunchKernelEx +
// CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION): each block records its rank in the
// cluster, the cluster size, and its neighbour's value read through
// distributed shared memory -- all different without the cluster launch.
extern "C" __global__ void kc_fixture_cluster(unsigned int* out) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ unsigned int v;
    if (threadIdx.x == 0) v = blockIdx.x * 7u + 1u;
    cl.sync();
    const unsigned int rank = cl.block_rank(), nb = cl.num_blocks();
    const unsigned int* peer = cl.map_shared_rank(&v, (rank + 1) % nb);
    if (threadIdx.x == 0) out[blockIdx.x] = (rank << 24) | (nb << 16) | (*peer & 0xFFFFu);
    cl.sync();
}

// A cooperative launch (grid-wide synchronisation): every block publishes a
// value, the whole grid synchronises, then each block reads its neighbour's.
// Launched without the cooperative attribute, grid.sync() is not allowed.
extern "C" __global__ void kc_fixture_coop(unsigned int* stage, unsigned int* out) {
    namespace cg = cooperative_groups;
    cg::grid_group g = cg::this_grid();
    if (threadIdx.x == 0) stage[blockIdx.x] = blockIdx.x * 13u + 5u;
    g.sync();
    if (threadIdx.x == 0) out[blockIdx.x] = stage[(blockIdx.x + 1) % gridDim.x] ^ 0xA5A5u;
}
