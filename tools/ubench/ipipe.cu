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
#include <cstdint>
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
    // operands in registers (a kernel parameter used under a predicate is
    // otherwise re-read from the constant bank inside the predicated block)
    unsigned yr = y ^ *(volatile unsigned *)&out[0], xr = x ^ *(volatile unsigned *)&out[1];
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
            if constexpr (V == 13) e[i] = e[i] * xr + yr;                              // IMAD
            if constexpr (V == 14) e[i] = __byte_perm(e[i], xr, 0x5410u + i);          // PRMT
            if constexpr (V == 15) e[i] = __umulhi(e[i], xr) ^ (unsigned)i;            // IMAD.HI (+LOP3?)
            if constexpr (V == 16) {                                                  // 1 ALU : 1 IMAD
                if (i & 1) e[i] = __viaddmax_u16x2(e[i], xr, yr);
                else e[i] = e[i] * xr + yr;
            }
            if constexpr (V == 17) {                                                  // 2 ALU : 1 IMAD
                if (i % 3 != 2) e[i] = __viaddmax_u16x2(e[i], xr, yr);
                else e[i] = e[i] * xr + yr;
            }
            if constexpr (V == 18) e[i] = __viaddmin_u16x2(e[i], xr, yr);             // VIADDMNMX.U16x2 min
        }
        if constexpr (V == 12) {
            // six chains per mask word: one R2P sets P1..P6
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t nb = __umulhi(pm + (uint32_t)it, 0x9E3779B9u + 77u * i);
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    if (nb & (2u << q)) {
                        asm volatile("");
                        e[q] = __viaddmax_u16x2(e[q], xr + i, yr);
                    }
                }
            }
        }
        if constexpr (V == 10 || V == 11) {
            // the walk's mix: per position a mask word from the FMA pipe
            // (IMAD.HI), R2P into P1..P4, four predicated VIADDMNMX.U16x2 on
            // four chains (V == 11: the same without predicates)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t nb = __umulhi(pm + (uint32_t)it, 0x9E3779B9u + 77u * i);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (V == 11 || (nb & (2u << q))) {
                        asm volatile("");
                        e[q] = __viaddmax_u16x2(e[q], xr + i, yr);
                    }
                }
            }
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
void run(const char *name, const char *pipe, unsigned *d, int sms, int ctas_per_sm = 4)
{
    const int iters = 1 << 16, threads = 512, blocks = sms * ctas_per_sm;
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
        rate += (double)cnt[s] * threads / 32 * iters * (V == 12 ? 48 : V == 10 || V == 11 ? 32 : 8) / (4 * w);
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
    // walk mix: the rate printed counts the VIADDMNMX.U16x2 only (32 per
    // iteration: 8 positions x 4 chains), next to 8 R2P and 8 IMAD.HI
    run<10>("walk: R2P + 4 @P VIADDMNMX", "mix", d, sms);
    run<11>("walk without predicates", "mix", d, sms);
    // 4 warps per SMSP (one 512-thread CTA per SM), as the lb kernel runs
    run<10>("walk R2P, 4 warps/SMSP", "mix", d, sms, 1);
    run<11>("walk no pred, 4 warps/SMSP", "mix", d, sms, 1);
    run<0>("VIADDMNMX.U16x2 4w/SMSP", "alu", d, sms, 1);
    run<12>("walk 6 chains per R2P", "mix", d, sms);
    run<12>("walk 6 chains, 4w/SMSP", "mix", d, sms, 1);
    // round 2b: the job-pair heads' mix (FMA-pipe multiply-adds beside the ALU ops)
    run<13>("IMAD", "fma", d, sms);
    run<14>("PRMT", "alu?", d, sms);
    run<15>("IMAD.HI", "fma", d, sms);
    run<16>("VIADDMNMX|IMAD 1:1", "mix", d, sms);
    run<17>("VIADDMNMX|IMAD 2:1", "mix", d, sms);
    run<18>("VIADDMNMX.U16x2 (min)", "alu", d, sms);
    return 0;
}
