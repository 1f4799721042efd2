// Throughput of the walk's candidate integer instructions on sm_100a:
// each thread runs 8 independent dependency chains, 4096 steps.
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(unsigned *out, unsigned x, unsigned y, int iters)
{
    unsigned e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = threadIdx.x * (i + 1);
    unsigned pm = threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        x ^= it; y += it;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (V == 0) e[i] = __viaddmax_s16x2(e[i], x, y);             // VIADDMNMX.S16x2
            if constexpr (V == 1) e[i] = (unsigned)__viaddmax_s32((int)e[i], (int)x, (int)y); // VIADDMNMX
            if constexpr (V == 2) e[i] = (unsigned)max((int)e[i], (int)y);         // VIMNMX
            if constexpr (V == 3) e[i] = e[i] + x;                                 // IADD / IMAD.IADD
            if constexpr (V == 4) e[i] = (unsigned)max((int)(e[i] + x), (int)y);   // add + max
            if constexpr (V == 5) e[i] = __vmaxs2(e[i] , y);
            if constexpr (V == 8) e[i] = __vimax3_s16x2(e[i], x, y);                // VIMNMX3.S16x2
            if constexpr (V == 9) e[i] = __vimax3_s32((int)e[i], (int)x, (int)y);      // VIMNMX3                       // VIMNMX.S16x2
            if constexpr (V == 6) e[i] = e[i] ^ (x + i);                           // LOP3
            if constexpr (V == 7) { if ((pm >> i) & 1) e[i] = __viaddmax_s16x2(e[i], x, y); } // predicated
        }
        pm = pm * 1664525u + 1013904223u;
    }
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += e[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int V>
void run(const char *name, unsigned *d, int sms)
{
    const int iters = 4096, threads = 512, blocks = sms * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<V><<<blocks, threads>>>(d, 3, 5, iters);
    cudaEventRecord(a);
    k<V><<<blocks, threads>>>(d, 3, 5, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads / 32 * iters * 8; // warp-instructions of the op
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-22s %.3f ms  %.3f warp-ops/clk/SMSP\n", name, ms, ops / cyc / (sms * 4));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *d;
    cudaMalloc(&d, sizeof(unsigned) * sms * 4 * 512);
    run<0>("VIADDMNMX.S16x2", d, sms);
    run<1>("VIADDMNMX", d, sms);
    run<2>("VIMNMX", d, sms);
    run<3>("IADD", d, sms);
    run<4>("add+max", d, sms);
    run<5>("VIMNMX.S16x2", d, sms);
    run<6>("LOP3", d, sms);
    run<7>("@P VIADDMNMX.S16x2", d, sms);
    run<8>("VIMNMX3.S16x2", d, sms);
    run<9>("VIMNMX3", d, sms);
    return 0;
}
