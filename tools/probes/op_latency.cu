// Dependent-latency probe for the integer ops on K1's XXH64 chain (one warp,
// 1,024 dependent ops per measurement, clock64): which op makes a round cost
// ~30 cycles when the chain is SHF -> IMAD -> IMAD -> IMAD.WIDE?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/op_latency tools/probes/op_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 1024

template <int OP>
__global__ void lat(uint32_t seed, uint32_t* out, long long* cyc) {
    uint32_t a = seed + threadIdx.x, b = seed * 3u + 1u;
    uint64_t w = ((uint64_t)b << 32) | a;
    const uint32_t k = 0x85EBCA87u;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(k), "r"(b));           // IMAD
        if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(k), "r"(b));           // IMAD.HI
        if (OP == 2) {                                                                               // IMAD.WIDE (lo feeds)
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"((uint32_t)w), "r"(k));
        }
        if (OP == 3) asm volatile("shf.l.wrap.b32 %0, %0, %1, 31;" : "+r"(a) : "r"(b));               // SHF
        if (OP == 4) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));                          // IADD3
        if (OP == 5) {                                                                               // IMAD.WIDE (hi feeds)
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w) : "r"((uint32_t)(w >> 32)), "r"(k));
        }
        if (OP == 6) {  // SHF -> IMAD alternating (cross-pipe)
            asm volatile("shf.l.wrap.b32 %0, %0, %1, 31;\n\tmad.lo.u32 %0, %0, %2, %1;" : "+r"(a) : "r"(b), "r"(k));
        }
        if (OP == 7) {  // 64-bit mul.lo.u64 (emulated)
            asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(w) : "l"(0x9E3779B185EBCA87ULL));
        }
        if (OP == 8) {  // mad.lo.cc + madc.hi on the lo result
            uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
            asm volatile("mad.lo.cc.u32 %0, %0, %2, %1;\n\tmadc.hi.u32 %1, %0, %2, %1;" : "+r"(lo), "+r"(hi) : "r"(k));
            w = ((uint64_t)hi << 32) | lo;
        }
        if (OP == 9) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a) : "r"(b));                          // LOP3
        if (OP == 10) asm volatile("mul.lo.u32 %0, %0, 0x85EBCA87;" : "+r"(a));                       // IMAD imm
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ (uint32_t)w ^ (uint32_t)(w >> 32);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(const char* name, uint32_t* d_out, long long* d_cyc) {
    lat<OP><<<1, 32>>>(7u, d_out, d_cyc);
    lat<OP><<<1, 32>>>(7u, d_out, d_cyc);
    long long c = 0;
    cudaMemcpy(&c, d_cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const int per = (OP == 6 || OP == 8) ? 2 : 1;
    printf("%-34s %6.2f cycles per op\n", name, (double)c / (N * per));
}

int main() {
    uint32_t* d_out;
    long long* d_cyc;
    cudaMalloc(&d_out, 4096);
    cudaMalloc(&d_cyc, 64);
    run<0>("IMAD (mad.lo.u32)", d_out, d_cyc);
    run<10>("IMAD imm (mul.lo.u32)", d_out, d_cyc);
    run<1>("IMAD.HI (mad.hi.u32)", d_out, d_cyc);
    run<2>("IMAD.WIDE lo->a", d_out, d_cyc);
    run<5>("IMAD.WIDE hi->a", d_out, d_cyc);
    run<3>("SHF.L.W", d_out, d_cyc);
    run<4>("IADD3", d_out, d_cyc);
    run<9>("LOP3", d_out, d_cyc);
    run<6>("SHF<->IMAD alternating (per op)", d_out, d_cyc);
    run<7>("mul.lo.u64", d_out, d_cyc);
    run<8>("mad.lo.cc/madc.hi (per op)", d_out, d_cyc);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
