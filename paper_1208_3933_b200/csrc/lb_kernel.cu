// lb_kernel.cu — batched Lageweg-Lenstra-Rinnooy Kan two-machine bound on sm_100a.
//
// Computes, for every node of a pool, the LB of Fig. 3 with the
// readings R1-R6 of DESIGN.md §3.  Design:
//   * one thread per sub-problem, as the paper maps it, 32 nodes per
//     warp; every table read in the pair walk is then warp-uniform (broadcast);
//   * the per-couple tables (Johnson-with-lags order with each job's constants
//     folded into an 8-byte record) are staged into shared memory by TMA bulk
//     copies (cp.async.bulk + mbarrier), one couple group at a time when the
//     whole set exceeds shared memory (200x20: 2 groups);
//   * per warp, the unscheduled sets of its 32 nodes live in a transposed
//     bitset U[job] (bit L = job unscheduled in lane L's node), built from
//     coalesced reads of the prefix records;
//   * the walk of Fig. 3 lines 08-17 is carried in the (u, w) form
//         u <- max(u, w + c1_j);  w <- w + c2_j      (if j unscheduled)
//     two integer ops per update (VIADDMNMX + IADD), exact in int32.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "fsp_internal.h"

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// TMA 1-D bulk copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Issue the bulk copies of `bytes` (multiple of 16) in <= 32 KB pieces.
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    const uint32_t piece = 32768;
    for (uint32_t off = 0; off < bytes; off += piece) {
        uint32_t b = bytes - off < piece ? bytes - off : piece;
        bulk_g2s(static_cast<uint8_t *>(dst) + off, static_cast<const uint8_t *>(src) + off, b, bar);
    }
}

struct LbArgs {
    const uint8_t *tables; // groups x group_bytes
    const uint16_t *ptm16; // [n][mp] u16, ptm_bytes
    const uint16_t *prefix;
    const int32_t *depth;
    int32_t *lb_out;
    int *err;
    long long pool;
    unsigned long long group_bytes;
    int ptm_bytes;
    int warp_bytes;
    int groups, ppg;       // couple groups, couples per group
    int n, m, P, mp;       // mp = PTM row stride in u16 (even)
    int stride;
    int kl_bytes;          // couple-id header bytes of a group blob
};

template <int MAXM>
__global__ void __launch_bounds__(256) lb_kernel(const LbArgs a)
{
    extern __shared__ __align__(128) uint8_t smem[];
    const int n = a.n, m = a.m;
    uint8_t *s_tab = smem;
    const uint16_t *s_ptm = reinterpret_cast<const uint16_t *>(smem + a.group_bytes);
    uint64_t *s_bar = reinterpret_cast<uint64_t *>(smem + a.group_bytes + a.ptm_bytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    uint8_t *s_warp = smem + a.group_bytes + a.ptm_bytes + 16 + (size_t)warp * a.warp_bytes;
    uint32_t *U = reinterpret_cast<uint32_t *>(s_warp);
    const int ubytes = ((n * 4) + 15) & ~15;
    int *Rs = reinterpret_cast<int *>(s_warp + ubytes); // [MAXM][32] heads
    int *Ts = Rs + MAXM * 32;                            // [MAXM][32] tail + load

    auto group_size = [&](int g) {
        int np = a.P - g * a.ppg;
        return np < a.ppg ? np : a.ppg;
    };
    auto group_blob = [&](int g) {
        return (uint32_t)((a.kl_bytes + (size_t)group_size(g) * n * sizeof(fsp_rec) + 15) & ~size_t(15));
    };

    // ---- stage PTM + the first couple group (TMA bulk, one mbarrier) ----
    if (threadIdx.x == 0) {
        mbar_init(s_bar, 1);
        uint32_t gb = group_blob(0);
        mbar_expect_tx(s_bar, gb + (uint32_t)a.ptm_bytes);
        bulk_copy(s_tab, a.tables, gb, s_bar);
        bulk_copy(const_cast<uint16_t *>(s_ptm), a.ptm16, (uint32_t)a.ptm_bytes, s_bar);
    }
    __syncthreads();
    uint32_t phase = 0;
    mbar_wait(s_bar, phase);
    phase ^= 1;
    int resident = 0;

    const long long ntiles = (a.pool + 31) >> 5;
    const long long nchunks = (ntiles + W - 1) / W;
    const uint32_t lanebit = 1u << lane;

    for (long long chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
        const long long tile = chunk * W + warp;
        const long long node = tile * 32 + lane;
        const bool has = node < a.pool;
        bool bad = false;

        // ---------------- a1: node ingest (depth, scheduled set) ----------------
        int d = 0;
        if (has) {
            d = a.depth[node];
            if (d < 0 || d > n || d > a.stride) {
                bad = true;
                d = 0;
            }
        }
        const uint32_t valid = __ballot_sync(0xffffffffu, has);
        for (int j = lane; j < n; j += 32) U[j] = valid;
        __syncwarp();
        // coalesced pass over the 32 prefix records: clear the scheduled bits
        for (int L = 0; L < 32; ++L) {
            const int dL = __shfl_sync(0xffffffffu, d, L);
            if (dL == 0) continue;
            const uint16_t *row = a.prefix + (size_t)(tile * 32 + L) * a.stride;
            for (int i = lane; i < dL; i += 32) {
                const uint32_t job = row[i];
                if (job < (uint32_t)n) U[job] &= ~(1u << L);
            }
            __syncwarp();
        }

        // prefix completion times C_k, one node per lane
        int C[MAXM];
#pragma unroll
        for (int k = 0; k < MAXM; ++k) C[k] = 0;
        {
            const uint16_t *row = a.prefix + (size_t)(has ? node : 0) * a.stride;
            for (int i = 0; i < d; ++i) {
                uint32_t job = row[i];
                if (job >= (uint32_t)n) {
                    bad = true;
                    job = 0;
                }
                const uint32_t *pr = reinterpret_cast<const uint32_t *>(s_ptm + job * a.mp);
                int prev = 0;
#pragma unroll
                for (int k2 = 0; k2 < (MAXM + 1) / 2; ++k2) {
                    const uint32_t w2 = 2 * k2 < m ? pr[k2] : 0u;
                    if (2 * k2 < m) {
                        C[2 * k2] = max(C[2 * k2], prev) + (int)(w2 & 0xffffu);
                        prev = C[2 * k2];
                    }
                    if (2 * k2 + 1 < MAXM && 2 * k2 + 1 < m) {
                        C[2 * k2 + 1] = max(C[2 * k2 + 1], prev) + (int)(w2 >> 16);
                        prev = C[2 * k2 + 1];
                    }
                }
            }
        }

        // ---------------- a2/a3: heads R_k, tails Q_l, loads L_l ----------------
        // r_j0 = C_0, r_jk = max(C_k, r_j,k-1 + p_j,k-1) (R3); R_k = min over
        // unscheduled j (R5); q_jl = sum_{i>l} p_ji, Q_l = min (R4); and the
        // remaining load L_l = sum_j p_jl that closes the (u, w) walk.
        int R[MAXM], Q[MAXM], Ld[MAXM];
#pragma unroll
        for (int k = 0; k < MAXM; ++k) {
            R[k] = INT_MAX;
            Q[k] = INT_MAX;
            Ld[k] = 0;
        }
        int cnt = 0;
        for (int j = 0; j < n; ++j) {
            const uint32_t uj = U[j];
            if (uj == 0) continue; // scheduled in every node of this warp
            const int act = (uj >> lane) & 1;
            const int nm = act ? 0 : INT_MAX;
            cnt += act;
            const uint32_t *pr = reinterpret_cast<const uint32_t *>(s_ptm + j * a.mp);
            int p[MAXM];
#pragma unroll
            for (int k2 = 0; k2 < (MAXM + 1) / 2; ++k2) {
                const uint32_t w2 = 2 * k2 < m ? pr[k2] : 0u;
                p[2 * k2] = (int)(w2 & 0xffffu);
                if (2 * k2 + 1 < MAXM) p[2 * k2 + 1] = (int)(w2 >> 16);
            }
            int r = C[0];
            R[0] = min(R[0], r | nm);
#pragma unroll
            for (int k = 1; k < MAXM; ++k) {
                if (k < m) {
                    r = max(C[k], r + p[k - 1]);
                    R[k] = min(R[k], r | nm);
                }
            }
            int q = 0;
#pragma unroll
            for (int l = MAXM - 1; l >= 0; --l) {
                if (l < m) {
                    Q[l] = min(Q[l], q | nm);
                    q += p[l];
                    Ld[l] += act * p[l];
                }
            }
        }
        if (has && cnt != n - d) bad = true; // repeated or out-of-range job
        if (cnt == 0) {                       // R6: complete schedule
#pragma unroll
            for (int k = 0; k < MAXM; ++k) {
                R[k] = C[k];
                Q[k] = 0;
                Ld[k] = 0;
            }
        }
#pragma unroll
        for (int k = 0; k < MAXM; ++k) {
            if (k < m) {
                Rs[k * 32 + lane] = R[k];
                Ts[k * 32 + lane] = Q[k] + Ld[k];
            }
        }
        if (bad) atomicOr(a.err, 1);
        __syncwarp();

        // ---------------- a4/a5: couple walks (Fig. 3 lines 03-19) ----------------
        int lb = 0; // R1
        const bool ascending = resident == 0;
        for (int gi = 0; gi < a.groups; ++gi) {
            const int g = ascending ? gi : a.groups - 1 - gi;
            if (g != resident) {
                __syncthreads(); // every warp is done with the resident group
                if (threadIdx.x == 0) {
                    fence_proxy_async();
                    const uint32_t gb = group_blob(g);
                    mbar_expect_tx(s_bar, gb);
                    bulk_copy(s_tab, a.tables + (size_t)g * a.group_bytes, gb, s_bar);
                }
                mbar_wait(s_bar, phase);
                phase ^= 1;
                resident = g;
            }
            if (valid == 0) continue;
            const uint32_t *kl = reinterpret_cast<const uint32_t *>(s_tab);
            const fsp_rec *recs = reinterpret_cast<const fsp_rec *>(s_tab + a.kl_bytes);
            const int np = group_size(g);
            const char *ub = reinterpret_cast<const char *>(U);
            for (int pl = 0; pl < np; ++pl) {
                const uint32_t kv = kl[pl];
                const int k = kv & 0xffff, l = kv >> 16;
                int u = Rs[l * 32 + lane]; // timeOnM2 starts at RM min of M2 (line 07)
                int w = Rs[k * 32 + lane]; // timeOnM1 starts at RM min of M1 (line 06)
                const fsp_rec *rp = recs + (size_t)pl * n;
#pragma unroll 8
                for (int i = 0; i < n; ++i) {
                    const fsp_rec r = rp[i];
                    const uint32_t msk =
                        *reinterpret_cast<const uint32_t *>(ub + (r.meta & 0xffff));
                    if (msk & lanebit) { // line 10: job not yet scheduled
                        u = max(u, w + r.c1);   // lines 11-15, (u, w) form
                        w += (r.meta >> 16);
                    }
                }
                lb = max(lb, u + Ts[l * 32 + lane]); // lines 18-19
            }
        }
        if (has) a.lb_out[node] = lb;
        __syncwarp();
    }
}

template <int MAXM>
int launch(const fsp_instance *inst, const LbArgs &a, cudaStream_t s)
{
    const fsp_lb_plan &pl = inst->plan;
    lb_kernel<MAXM><<<pl.grid, pl.warps * 32, pl.smem_bytes, s>>>(a);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "lb_kernel launch");
}

template <int MAXM>
int configure(fsp_instance *inst)
{
    fsp_lb_plan &pl = inst->plan;
    cudaError_t e = cudaFuncSetAttribute(lb_kernel<MAXM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pl.smem_bytes);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "cudaFuncSetAttribute");
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lb_kernel<MAXM>, pl.warps * 32,
                                                      pl.smem_bytes);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "occupancy");
    if (per_sm < 1) return fsp_fail(FSP_ERANGE, "lb kernel does not fit on an SM");
    pl.ctas_per_sm = per_sm;
    pl.grid = pl.num_sms * per_sm;
    return FSP_OK;
}

} // namespace

static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Choose the machine specialisation, couple groups and CTA shape so that one
// couple group + PTM + per-warp scratch fit the opt-in shared memory.
int fsp_plan_lb(fsp_instance *inst)
{
    fsp_lb_plan &pl = inst->plan;
    const int n = inst->n, m = inst->m, P = inst->P;
    static const int maxms[] = {5, 8, 10, 16, 20, 32};
    pl.maxm = 0;
    for (int mm : maxms)
        if (m <= mm) {
            pl.maxm = mm;
            break;
        }
    if (!pl.maxm) return fsp_fail(FSP_ERANGE, "m too large");
    int dev = inst->device, optin = 0, sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "device attribute");
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "device attribute");
    pl.num_sms = sms;
    const int mp = (m + 1) & ~1;
    pl.ptm_bytes = align16((size_t)n * mp * 2);
    pl.warp_bytes = align16((size_t)n * 4) + 2 * (size_t)pl.maxm * 32 * 4;
    int want_warps = 8;
    if (const char *s = getenv("FSP_LB_WARPS")) want_warps = atoi(s);
    if (want_warps < 1) want_warps = 1;
    if (want_warps > 8) want_warps = 8;
    for (int W = want_warps; W >= 1; W /= 2) {
        for (int G = 1; G <= P; ++G) {
            const int ppg = (P + G - 1) / G;
            const int Greal = (P + ppg - 1) / ppg;
            const size_t gb = align16((size_t)ppg * 4) + (size_t)ppg * n * sizeof(fsp_rec);
            const size_t total = gb + pl.ptm_bytes + 16 + (size_t)W * pl.warp_bytes;
            if (total <= (size_t)optin) {
                pl.groups = Greal;
                pl.pairs_per_group = ppg;
                pl.warps = W;
                pl.group_bytes = align16(gb);
                pl.smem_bytes = pl.group_bytes + pl.ptm_bytes + 16 + (size_t)W * pl.warp_bytes;
                switch (pl.maxm) {
                case 5: return configure<5>(inst);
                case 8: return configure<8>(inst);
                case 10: return configure<10>(inst);
                case 16: return configure<16>(inst);
                case 20: return configure<20>(inst);
                default: return configure<32>(inst);
                }
            }
            if (ppg == 1) break;
        }
    }
    return fsp_fail(FSP_ERANGE, "instance tables do not fit in shared memory");
}

int fsp_launch_lb(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                  const int32_t *depth, int64_t pool, int32_t *lb_out, cudaStream_t s)
{
    const fsp_lb_plan &pl = inst->plan;
    LbArgs a;
    a.tables = inst->d_tables;
    a.ptm16 = inst->d_ptm16;
    a.prefix = prefix;
    a.depth = depth;
    a.lb_out = lb_out;
    a.err = inst->d_err;
    a.pool = pool;
    a.group_bytes = pl.group_bytes;
    a.ptm_bytes = (int)pl.ptm_bytes;
    a.warp_bytes = (int)pl.warp_bytes;
    a.groups = pl.groups;
    a.ppg = pl.pairs_per_group;
    a.n = inst->n;
    a.m = inst->m;
    a.P = inst->P;
    a.mp = (inst->m + 1) & ~1;
    a.stride = stride;
    a.kl_bytes = (int)align16((size_t)pl.pairs_per_group * 4);
    switch (pl.maxm) {
    case 5: return launch<5>(inst, a, s);
    case 8: return launch<8>(inst, a, s);
    case 10: return launch<10>(inst, a, s);
    case 16: return launch<16>(inst, a, s);
    case 20: return launch<20>(inst, a, s);
    default: return launch<32>(inst, a, s);
    }
}
