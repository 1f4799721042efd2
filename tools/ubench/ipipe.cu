// Issue rate of the integer instructions the LB walk and phase A use, on sm_100a
// (VERDICT r1 "measure the integer peaks").  Each thread runs 8 independent
// dependency chains; 4 CTAs x 512 threads per SM (64 warps, 16 per SMSP), so
// latency is hidden and the number is the pipe's throughput.  The SM clock
// during the run comes from clock64() deltas of every CTA's thread 0 divided
// by the CUDA-event time, so warp-instructions per cycle are per ACTUAL cycle.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ipipe ipipe.cu && ./ipipe
//
// Output: one line per variant: warp-instructions of the measured op per
// cycle per SMSP (1.0 = one per clock = the issue limit; 0.5 = a half-rate
// pipe), plus the same as lane-ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
#include <climits>
#include <algorithm>
#include <vector>

// per CTA: SM id, clock64 at start and end (clock64 is per SM: windows are
// taken per SM as max(end) - min(start) over its CTAs)
__device__ long long g_t0[148 * 8], g_t1[148 * 8];
__device__ int g_sm[148 * 8];

template <int V>
__global__ void __launch_bounds__(512) k(unsigned *out, unsigned x, unsigned y, int iters)
{
    unsigned e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = threadIdx.x * (i + 1);
    unsigned pm = threadIdx.x * 2654435761u;
    __syncthreads();
    long long c0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (V == 0) e[i] = __viaddmax_u16x2(e[i], x, y);               // VIADDMNMX.U16x2
            if constexpr (V == 1) e[i] = (unsigned)__viaddmax_s32((int)e[i], (int)x, (int)y);  // VIADDMNMX
            if constexpr (V == 2) e[i] = __vminu2(e[i], y);                           // VIMNMX.U16x2
            if constexpr (V == 3) e[i] = (unsigned)max((int)e[i], (int)y);           // VIMNMX
            if constexpr (V == 4) e[i] = e[i] + x + (unsigned)i;                      // IADD3
            if constexpr (V == 5) e[i] = (e[i] ^ x) & (y | (unsigned)i);              // LOP3
            if constexpr (V == 6) e[i] = __umulhi(e[i], x) + y;                       // IMAD.HI (FMA pipe)
            if constexpr (V == 7) {                                                   // predicated
                if ((pm >> (i + 1)) & 1) e[i] = __viaddmax_u16x2(e[i], x, y);
            }
            if constexpr (V == 8) {                                                   // 1 ALU : 1 FMA
                if (i & 1) e[i] = __viaddmax_u16x2(e[i], x, y);
                else e[i] = __umulhi(e[i], x) + y;
            }
            if constexpr (V == 9) e[i] = __vimax3_u16x2(e[i], x, y);                  // VIMNMX3.U16x2
        }
        if constexpr (V == 7) pm = (pm ^ (pm >> 7)) + e[0];
        x += 3;
    }
    __syncthreads();
    long long c1 = clock64();
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += e[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_t0[blockIdx.x] = c0;
        g_t1[blockIdx.x] = c1;
        g_sm[blockIdx.x] = (int)sm;
    }
}

template <int V>
void run(const char *name, const char *pipe, unsigned *d, int sms)
{
    const int iters = 1 << 16, threads = 512, blocks = sms * 4;
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
    static long long t0[148 * 8], t1[148 * 8];
    static int sm[148 * 8];
    cudaMemcpyFromSymbol(t0, g_t0, sizeof(long long) * blocks);
    cudaMemcpyFromSymbol(t1, g_t1, sizeof(long long) * blocks);
    cudaMemcpyFromSymbol(sm, g_sm, sizeof(int) * blocks);
    std::vector<long long> lo(sms, LLONG_MAX), hi(sms, LLONG_MIN);
    std::vector<int> cnt(sms, 0);
    for (int i = 0; i < blocks; ++i) {
        lo[sm[i]] = std::min(lo[sm[i]], t0[i]);
        hi[sm[i]] = std::max(hi[sm[i]], t1[i]);
        cnt[sm[i]]++;
    }
    // per SM: warp-instructions of the op / (4 SMSPs x window cycles)
    double rate = 0, win = 0;
    int used = 0;
    for (int s = 0; s < sms; ++s) {
        if (!cnt[s]) continue;
        const double w = (double)(hi[s] - lo[s]);
        rate += (double)cnt[s] * threads / 32 * iters * 8 / (4 * w);
        win += w;
        ++used;
    }
    rate /= used;
    win /= used;
    printf("%-24s %-4s %8.3f ms %6.0f MHz(win/event) %6.3f warp-instr/clk/SMSP %6.1f lane-ops/clk/SM\n",
           name, pipe, ms, win / (ms * 1e3), rate, rate * 128);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("# %s, %d SMs, sm_%d%d; 4 CTAs x 512 threads per SM, 8 chains/thread\n", p.name, sms,
           p.major, p.minor);
    unsigned *d;
    cudaMalloc(&d, sizeof(unsigned) * sms * 4 * 512);
    for (int w = 0; w < 20; ++w) k<0><<<sms * 4, 512>>>(d, 3, 5, 1 << 16); // clocks up
    cudaDeviceSynchronize();
    run<0>("VIADDMNMX.U16x2", "alu", d, sms);
    run<7>("@P VIADDMNMX.U16x2", "alu", d, sms);
    run<1>("VIADDMNMX", "alu", d, sms);
    run<2>("VIMNMX.U16x2", "alu", d, sms);
    run<3>("VIMNMX", "alu", d, sms);
    run<9>("VIMNMX3.U16x2", "alu", d, sms);
    run<4>("IADD3", "alu", d, sms);
    run<5>("LOP3", "alu", d, sms);
    run<6>("IMAD.HI+IADD3", "fma", d, sms);
    run<8>("VIADDMNMX.U16x2|IMAD.HI", "mix", d, sms);
    return 0;
}
