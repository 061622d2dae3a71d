// K1 round latency probe: cycles per XXH64 round for one chain per thread, one
// warp per SMSP (the sub-wave K1 case), for several formulations of the round.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/k1_round_probe tools/probes/k1_round_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define P1 0x9E3779B185EBCA87ULL
#define P2 0xC2B2AE3D27D4EB4FULL

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
__device__ __forceinline__ uint64_t r_plain(uint64_t acc, uint64_t x) { acc += x * P2; acc = rotl64(acc, 31); return acc * P1; }
__device__ __forceinline__ uint64_t r_fast(uint64_t acc, uint64_t x) {
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    uint64_t w;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(xl), "r"((uint32_t)P2), "l"(acc));
    const uint32_t t = xl * (uint32_t)(P2 >> 32) + xh * (uint32_t)P2;
    const uint32_t sl = (uint32_t)w, sh = (uint32_t)(w >> 32) + t;
    const uint32_t rh = __funnelshift_l(sl, sh, 31), rl = __funnelshift_l(sh, sl, 31);
    uint64_t w2;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(w2) : "r"(rl), "r"((uint32_t)P1));
    const uint32_t t2 = rl * (uint32_t)(P1 >> 32) + rh * (uint32_t)P1;
    return (w2 & 0xFFFFFFFFull) | ((uint64_t)((uint32_t)(w2 >> 32) + t2) << 32);
}
__device__ __forceinline__ uint64_t r_y(uint64_t y, uint64_t x) {
    const uint64_t p = x * P2;
    const uint32_t yl = (uint32_t)y, yh = (uint32_t)(y >> 32);
    const uint32_t rh = __funnelshift_l(yl, yh, 31), rl = __funnelshift_l(yh, yl, 31);
    uint64_t w;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(rl), "r"((uint32_t)P1), "l"(p));
    const uint32_t hi = (uint32_t)(w >> 32) + rl * (uint32_t)(P1 >> 32) + rh * (uint32_t)P1;
    return ((uint64_t)hi << 32) | (uint32_t)w;
}
// y form with the low/high halves as explicit carry-chain PTX (add.cc / addc)
__device__ __forceinline__ uint64_t r_ycc(uint64_t y, uint64_t x) {
    const uint64_t p = x * P2;
    const uint32_t yl = (uint32_t)y, yh = (uint32_t)(y >> 32);
    const uint32_t rh = __funnelshift_l(yl, yh, 31), rl = __funnelshift_l(yh, yl, 31);
    uint32_t lo, hi;
    const uint32_t c = rl * (uint32_t)(P1 >> 32) + rh * (uint32_t)P1 + (uint32_t)(p >> 32);
    asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.u32 %1, %2, %3, %5;"
        : "=r"(lo), "=r"(hi) : "r"(rl), "r"((uint32_t)P1), "r"((uint32_t)p), "r"(c));
    return ((uint64_t)hi << 32) | lo;
}

// the kernel's round (kc_kernels.cu ystep): chain SHF -> IMAD -> IMAD -> IMAD.WIDE
__device__ __forceinline__ uint64_t r_k(uint64_t y, uint64_t x) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh, yl, yh, plo, phi, rl, rh, t;\n\t"
        "mov.b64 {xl, xh}, %2;\n\tmov.b64 {yl, yh}, %3;\n\t"
        "mul.lo.u32 plo, xl, %4;\n\tmul.hi.u32 phi, xl, %4;\n\t"
        "mad.lo.u32 phi, xl, %5, phi;\n\tmad.lo.u32 phi, xh, %4, phi;\n\t"
        "shf.l.wrap.b32 rh, yl, yh, 31;\n\tshf.l.wrap.b32 rl, yh, yl, 31;\n\t"
        "mad.lo.u32 t, rh, %6, phi;\n\tmad.lo.u32 t, rl, %7, t;\n\t"
        "mad.lo.cc.u32 %0, rl, %6, plo;\n\tmadc.hi.u32 %1, rl, %6, t;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "l"(y), "r"((uint32_t)P2), "r"((uint32_t)(P2 >> 32)), "r"((uint32_t)P1), "r"((uint32_t)(P1 >> 32)));
    return ((uint64_t)hi << 32) | lo;
}
// IMAD.WIDE off the chain: hi = mul.hi(rl, P1lo) + t + carry(rl*P1lo + plo) as IADD3.X
__device__ __forceinline__ uint64_t r_h(uint64_t y, uint64_t x) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh, yl, yh, plo, phi, rl, rh, t, m, mh;\n\t"
        "mov.b64 {xl, xh}, %2;\n\tmov.b64 {yl, yh}, %3;\n\t"
        "mul.lo.u32 plo, xl, %4;\n\tmul.hi.u32 phi, xl, %4;\n\t"
        "mad.lo.u32 phi, xl, %5, phi;\n\tmad.lo.u32 phi, xh, %4, phi;\n\t"
        "shf.l.wrap.b32 rh, yl, yh, 31;\n\tshf.l.wrap.b32 rl, yh, yl, 31;\n\t"
        "mad.lo.u32 t, rh, %6, phi;\n\tmad.lo.u32 t, rl, %7, t;\n\t"
        "mul.hi.u32 mh, rl, %6;\n\tmul.lo.u32 m, rl, %6;\n\t"
        "add.cc.u32 %0, m, plo;\n\taddc.u32 %1, mh, t;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "l"(y), "r"((uint32_t)P2), "r"((uint32_t)(P2 >> 32)), "r"((uint32_t)P1), "r"((uint32_t)(P1 >> 32)));
    return ((uint64_t)hi << 32) | lo;
}
// carry from a compare: lo = mad.lo(rl, P1lo, plo); c = lo < plo; hi = mul.hi + t + c
__device__ __forceinline__ uint64_t r_c(uint64_t y, uint64_t x) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh, yl, yh, plo, phi, rl, rh, t, mh, c;\n\t.reg .pred q;\n\t"
        "mov.b64 {xl, xh}, %2;\n\tmov.b64 {yl, yh}, %3;\n\t"
        "mul.lo.u32 plo, xl, %4;\n\tmul.hi.u32 phi, xl, %4;\n\t"
        "mad.lo.u32 phi, xl, %5, phi;\n\tmad.lo.u32 phi, xh, %4, phi;\n\t"
        "shf.l.wrap.b32 rh, yl, yh, 31;\n\tshf.l.wrap.b32 rl, yh, yl, 31;\n\t"
        "mad.lo.u32 t, rh, %6, phi;\n\tmad.lo.u32 t, rl, %7, t;\n\t"
        "mul.hi.u32 mh, rl, %6;\n\tmad.lo.u32 %0, rl, %6, plo;\n\t"
        "setp.lt.u32 q, %0, plo;\n\tselp.u32 c, 1, 0, q;\n\t"
        "add.u32 t, t, c;\n\tadd.u32 %1, mh, t;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "l"(y), "r"((uint32_t)P2), "r"((uint32_t)(P2 >> 32)), "r"((uint32_t)P1), "r"((uint32_t)(P1 >> 32)));
    return ((uint64_t)hi << 32) | lo;
}
// mad.hi with t as addend, then the carry
__device__ __forceinline__ uint64_t r_d(uint64_t y, uint64_t x) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh, yl, yh, plo, phi, rl, rh, t, m, mh;\n\t"
        "mov.b64 {xl, xh}, %2;\n\tmov.b64 {yl, yh}, %3;\n\t"
        "mul.lo.u32 plo, xl, %4;\n\tmul.hi.u32 phi, xl, %4;\n\t"
        "mad.lo.u32 phi, xl, %5, phi;\n\tmad.lo.u32 phi, xh, %4, phi;\n\t"
        "shf.l.wrap.b32 rh, yl, yh, 31;\n\tshf.l.wrap.b32 rl, yh, yl, 31;\n\t"
        "mad.lo.u32 t, rh, %6, phi;\n\tmad.lo.u32 t, rl, %7, t;\n\t"
        "mad.hi.u32 mh, rl, %6, t;\n\tmul.lo.u32 m, rl, %6;\n\t"
        "add.cc.u32 %0, m, plo;\n\taddc.u32 %1, mh, 0;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "l"(y), "r"((uint32_t)P2), "r"((uint32_t)(P2 >> 32)), "r"((uint32_t)P1), "r"((uint32_t)(P1 >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

// IMAD.WIDE(rl, P1lo, {plo, phi}) with the rh*P1lo + rl*P1hi terms added after it (kernel ystep_h)
__device__ __forceinline__ uint64_t r_w(uint64_t y, uint64_t x) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh, yl, yh, plo, phi, rl, rh, a, b, h0;\n\t"
        "mov.b64 {xl, xh}, %2;\n\tmov.b64 {yl, yh}, %3;\n\t"
        "mul.lo.u32 plo, xl, %4;\n\tmul.hi.u32 phi, xl, %4;\n\t"
        "mad.lo.u32 phi, xl, %5, phi;\n\tmad.lo.u32 phi, xh, %4, phi;\n\t"
        "shf.l.wrap.b32 rh, yl, yh, 31;\n\tshf.l.wrap.b32 rl, yh, yl, 31;\n\t"
        "mad.lo.cc.u32 %0, rl, %6, plo;\n\tmadc.hi.u32 h0, rl, %6, phi;\n\t"
        "mul.lo.u32 a, rh, %6;\n\tmad.lo.u32 b, rl, %7, a;\n\tadd.u32 %1, h0, b;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "l"(y), "r"((uint32_t)P2), "r"((uint32_t)(P2 >> 32)), "r"((uint32_t)P1), "r"((uint32_t)(P1 >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

template <int V, int CH>
__global__ void probe(const uint64_t* __restrict__ in, uint64_t* out, long long* cyc, int rounds) {
    __shared__ uint64_t sx[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sx[i] = in[i];
    __syncthreads();
    uint64_t v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 7919ull + c;
    const uint64_t* p = sx + (threadIdx.x & 31);
    long long t0 = clock64();
    for (int t = 0; t < rounds; t += 32) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const uint64_t x = p[(u * 32 + t) & 4095];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (V == 0) v[c] = r_plain(v[c], x + c);
                if (V == 1) v[c] = r_fast(v[c], x + c);
                if (V == 2) v[c] = r_y(v[c], x + c);
                if (V == 3) v[c] = r_ycc(v[c], x + c);
                if (V == 4) v[c] = r_k(v[c], x + c);
                if (V == 5) v[c] = r_h(v[c], x + c);
                if (V == 6) v[c] = r_c(v[c], x + c);
                if (V == 7) v[c] = r_d(v[c], x + c);
                if (V == 8) v[c] = r_w(v[c], x + c);
            }
        }
    }
    long long t1 = clock64();
    uint64_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V, int CH>
void run(const char* name, uint64_t* in, uint64_t* out, long long* cyc, int threads) {
    const int rounds = 2048;
    probe<V, CH><<<148, threads>>>(in, out, cyc, rounds);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<V, CH><<<148, threads>>>(in, out, cyc, rounds);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    static uint64_t got[148 * 1024];
    // host reference for the y-form variants (V >= 2): y' = rotl(y, 31)*P1 + x*P2 with every x = 0x5a..5a
    bool same = true;
    if (V >= 2 && CH == 1) {
        cudaMemcpy(got, out, 148 * threads * 8, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 148 * threads && same; ++i) {
            uint64_t y = (uint64_t)(i % threads) * 7919ull;
            for (int r = 0; r < rounds; ++r) y = rotl64(y, 31) * P1 + 0x5a5a5a5a5a5a5a5aULL * P2;
            same = got[i] == y;
        }
    }
    long long c[148];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += c[i];
    avg /= 148;
    printf("%-34s threads/CTA %4d chains/thread %d: %6.1f cycles per round-step, kernel %.1f us%s\n", name, threads, CH,
           avg / rounds, ms * 1e3, same ? "" : "  RESULT DIFFERS");
}

int main() {
    uint64_t *in, *out;
    long long* cyc;
    cudaMalloc(&in, 4096 * 8);
    cudaMemset(in, 0x5a, 4096 * 8);
    cudaMalloc(&out, 148 * 1024 * 8);
    cudaMalloc(&cyc, 148 * 8);
    for (int th : {32, 64, 128, 256}) {
        run<0, 1>("plain 64-bit", in, out, cyc, th);
        run<1, 1>("r1 fast (mad.wide + funnel)", in, out, cyc, th);
        run<2, 1>("y form", in, out, cyc, th);
        run<3, 1>("y form, mad.lo.cc/madc.hi", in, out, cyc, th);
    }
    for (int th : {32, 128}) {
        run<2, 1>("y form", in, out, cyc, th);
        run<4, 1>("kernel round (IMAD.WIDE last)", in, out, cyc, th);
        run<2, 1>("y form", in, out, cyc, th);
        run<5, 1>("mul.hi + add.cc/addc", in, out, cyc, th);
        run<2, 1>("y form", in, out, cyc, th);
        run<6, 1>("mad.lo + setp carry", in, out, cyc, th);
        run<2, 1>("y form", in, out, cyc, th);
        run<7, 1>("mad.hi(t) + add.cc/addc", in, out, cyc, th);
        run<2, 1>("y form", in, out, cyc, th);
        run<8, 1>("IMAD.WIDE(plo,phi) + late adds", in, out, cyc, th);
    }
    run<2, 2>("y form", in, out, cyc, 128);
    run<2, 4>("y form", in, out, cyc, 128);
    run<3, 2>("y form, mad.lo.cc/madc.hi", in, out, cyc, 128);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
