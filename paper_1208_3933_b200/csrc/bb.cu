// bb.cu — device-resident B&B for the permutation FSP.
//
// The four operators of §II-A with the paper's forward branching
// and elimination LB >= incumbent (R9), all on the device:
//   selection  (a9)  the top B open nodes of a device stack (deepest-first
//                    batches replace the paper's host best-first list, R10);
//   branching  (a7)  lazy: a popped parent generates its next K children
//                    (prefix + j, j unscheduled), taken in ascending
//                    order of the idle time j adds (R19), and, if it has more,
//                    goes back on the stack below them with an advanced cursor
//                    (bounded memory); each child's
//                    completion times come from its parent's in one step;
//   bounding   (a1-a5) the LB kernel on the child pool with the sparse-walk plan
//                    (children of nearby parents share most of their
//                    unscheduled set), pool size read on the device;
//   elimination (a6) prune + scan + scatter: survivors (LB < incumbent) are
//                    stream-compacted onto the stack, each parent's children
//                    in descending (LB, idle, j) so its best child is on top
//                    (best-first among siblings, R10/R19), parents
//                    whose stored LB reached the incumbent are dropped at pop;
//                    leaves (depth >= n-1: LB is the exact makespan, R6/P4) feed
//                    a packed (makespan, index) atomicMin and commit_kernel
//                    adopts the best one with its permutation (a8).
// One small status read per iteration is the only host round trip.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "fsp_internal.h"

namespace {

constexpr int kScanThreads = 1024;
constexpr int kPruneThreads = 1024;
constexpr unsigned long long kNoCand = ~0ull;

struct BBStatus {
    long long children;  // children bounded this iteration
    long long kept;      // popped parents pushed back (more children to come)
    long long survivors; // children pushed onto the stack
    int incumbent;       // current incumbent (INT_MAX = none)
    int improved;        // this rank's incumbent improved this iteration
};

// Open nodes, structure of arrays: prefix, depth, completion times C[m],
// cursor (children already generated), LB from when the node was bounded,
// key (idle << 12 | j) of the last child generated.
struct Nodes {
    uint16_t *pf = nullptr;
    int32_t *dp = nullptr, *C = nullptr, *cur = nullptr, *lb = nullptr;
    long long *kl = nullptr; // key of the last child generated (-1: none yet)
};

struct BBState {
    const fsp_instance *inst;
    int rank, world, n, m, stride, K;
    int64_t dive_iters;   // iterations of the first single-parent dive
    double beam;          // a descent of n levels may fill this fraction of the stack
    int64_t cap;          // stack capacity (nodes)
    int64_t base, size;   // open nodes live in [base, size)
    int64_t ccap;         // children per iteration (buffer capacity)
    int64_t kcap;         // parents per iteration
    Nodes st, kp, ch;     // stack, kept parents (scratch), children
    unsigned long long *ch_key; // per child: (idle << 12) | j (R19 tie key)
    uint16_t *ch_uf;      // per child: its unscheduled jobs (n - depth entries, stride)
    uint16_t *ppf;        // lazy rows (with ch_uf): the popped parents' rows [kcap][stride]
    int32_t *ch_par;      // lazy rows: child -> parent index in the batch
    int32_t *ord;         // child slot -> child record, siblings by descending (LB, key)
    int32_t *d_maxnp;     // largest |S| among this iteration's expanded parents
    int32_t *d_famflag;   // 1: the family kernel bounds this iteration's children
    int64_t *d_count_sparse; // children for the lb kernel (0 when the family kernel runs)
    bool family;          // sibling-incremental bounding enabled (n <= 256)
    long long *plan;      // per parent: (keep << 32) | children now
    int64_t *off;         // exclusive scan of plan; off[B] = (kept << 32) | children
    int64_t *d_count;     // children this iteration (LB pool size)
    int64_t *boff;        // survivor offsets per prune block
    long long *tsum;      // device_scan scratch: tile sums and their offsets
    int64_t *toff;
    int32_t *bcnt;
    int32_t *d_inc;       // incumbent makespan (pruning threshold)
    unsigned long long *d_cand;
    long long *d_packed;  // (own best << 32) | rank for the MIN all-reduce
    long long *d_scratch;
    int32_t *d_perm;      // this rank's best permutation
    unsigned long long *d_stats; // [pruned, leaves]
    BBStatus *d_status, *h_status;
    int64_t last_children; // children of the last iteration (still in ch)
    cudaEvent_t ev_in, ev_out; // ordering against a caller's stream (fsp_bb_step)
    int order;            // 1: best-first children (R19); 0 (FSP_BB_ORDER=0, A/B): job order, no dive
    bool timing;          // FSP_BB_TIMING: sum the iterations' device time
    cudaEvent_t ev_t0, ev_t1;
    double gpu_ms;
    cudaStream_t stream;
    bool own_stream, sparse;
    fsp_bb_stats stats;
    int have;             // this rank holds a permutation ...
    int32_t perm_ms;      // ... of this makespan (the incumbent may be lower: adopted)
    int32_t initial_inc;  // initial_ub + 1 (saturating)
};

__device__ __forceinline__ long long warp_excl_scan64(long long v, int lane, long long &total)
{
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// Block-wide exclusive scan of one int64 per thread (blockDim multiple of 32).
__device__ __forceinline__ long long block_excl_scan(long long v, long long &total)
{
    __shared__ long long wsum[32];
    __shared__ long long s_tot;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long wt;
    const long long ex = warp_excl_scan64(v, lane, wt);
    if (lane == 31) wsum[warp] = wt;
    __syncthreads();
    if (warp == 0) {
        const long long x = lane < nw ? wsum[lane] : 0;
        long long t;
        const long long e = warp_excl_scan64(x, lane, t);
        if (lane < nw) wsum[lane] = e;
        if (lane == 0) s_tot = t;
    }
    __syncthreads();
    const long long r = ex + wsum[warp];
    total = s_tot;
    __syncthreads(); // wsum / s_tot are reused by the next call
    return r;
}

// Exclusive scan of N items; out[N] = total.  Items are int64 (in64) or int32
// (in32).  If count_out: *count_out = low 32 bits of the total.
// Large N: scan_local_kernel scans 1024-item tiles in parallel and writes tile
// sums, scan_kernel (one block) scans the sums, scan_add_kernel adds them back.
__global__ void __launch_bounds__(kScanThreads)
    scan_kernel(const long long *in64, const int32_t *in32, int64_t N, int64_t *out,
                int64_t *count_out)
{
    long long carry = 0;
    for (int64_t t0 = 0; t0 < N; t0 += blockDim.x) {
        const int64_t i = t0 + threadIdx.x;
        long long v = 0;
        if (i < N) v = in64 ? in64[i] : (long long)in32[i];
        long long tot;
        const long long ex = block_excl_scan(v, tot);
        if (i < N) out[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) {
        out[N] = carry;
        if (count_out) *count_out = carry & 0xffffffffll;
    }
}

__global__ void __launch_bounds__(kScanThreads)
    scan_local_kernel(const long long *in64, const int32_t *in32, int64_t N, int64_t *out,
                      long long *tile_sums)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long v = 0;
    if (i < N) v = in64 ? in64[i] : (long long)in32[i];
    long long tot;
    const long long ex = block_excl_scan(v, tot);
    if (i < N) out[i] = ex;
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads)
    scan_add_kernel(int64_t N, int64_t *out, const int64_t *tile_off)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) out[i] += tile_off[blockIdx.x];
}

__global__ void scan_total_kernel(int64_t N, int64_t *out, const int64_t *tile_off, int64_t tiles,
                                  int64_t *count_out)
{
    out[N] = tile_off[tiles];
    if (count_out) *count_out = tile_off[tiles] & 0xffffffffll;
}

// Selection (a9) bookkeeping: per popped parent, children to generate now
// (at most K) and whether it stays open.  A parent whose LB (bounded when it
// was a child) has reached the incumbent since is eliminated here (R9).
__global__ void plan_kernel(Nodes st, int64_t first, int64_t B, int n, int K, const int32_t *inc_dev,
                            long long *plan, unsigned long long *stats, int32_t *maxnp)
{
    const int inc = *inc_dev;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int dropped = 0, np = 0;
    if (p < B) {
        const int64_t i = first + p;
        long long g = 0, keep = 0;
        if (st.lb[i] < inc) {
            np = n - st.dp[i];
            const int r = np - st.cur[i];
            g = r < K ? r : K;
            keep = r > g;
        } else {
            dropped = 1;
        }
        plan[p] = (keep << 32) | g;
    }
    np = __reduce_max_sync(0xffffffffu, (unsigned)np);
    if ((threadIdx.x & 31) == 0 && np) atomicMax(maxnp, np);
    const unsigned b = __ballot_sync(0xffffffffu, dropped);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(&stats[0], (unsigned long long)__popc(b));
}

// Bounding route: the family kernel (sibling-incremental, family.cu) when
// every expanded parent has at most 32 unscheduled jobs, else the lb kernel.
__global__ void route_kernel(const int32_t *maxnp, const int64_t *count, int family, int32_t *flag,
                             int64_t *count_sparse)
{
    const int fam = family && *maxnp <= 32;
    *flag = fam;
    *count_sparse = fam ? 0 : *count;
}

// uint4 q of child row = its parent's row (d entries) with job x at position d
// (rows padded with 0xffff); rows are 16-byte aligned (stride multiple of 8).
__device__ __forceinline__ uint4 child_vec(const uint4 *prow4, int d, int x, int q)
{
    const int d8 = (d + 7) >> 3;
    uint4 v = q < d8 ? prow4[q] : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    if (q == (d >> 3)) {
        uint32_t *w4 = reinterpret_cast<uint32_t *>(&v);
        const int t8 = d & 7;
        uint32_t &wd = w4[t8 >> 1];
        wd = (t8 & 1) ? ((wd & 0xffffu) | ((uint32_t)x << 16)) : ((wd & 0xffff0000u) | (uint32_t)x);
    }
    return v;
}

// Child prefix rows on demand (lazy mode: expand keeps the parents' rows
// only; the bounding reads unscheduled lists): debug hook.
__global__ void materialize_kernel(const uint16_t *__restrict__ ppf, const int32_t *__restrict__ ch_par,
                                   const unsigned long long *__restrict__ ch_key, const int32_t *__restrict__ cdp,
                                   int64_t cnt, int stride, uint16_t *cpf)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < cnt; c += warps) {
        const int d = cdp[c] - 1, x = (int)(ch_key[c] & 0xfffu);
        const uint4 *prow4 = reinterpret_cast<const uint4 *>(ppf + (size_t)ch_par[c] * stride);
        uint4 *crow4 = reinterpret_cast<uint4 *>(cpf + (size_t)c * stride);
        for (int q = lane; q < (stride >> 3); q += 32) crow4[q] = child_vec(prow4, d, x, q);
    }
}

// Branching (a7): one warp per parent; its unscheduled jobs of ascending
// (idle, j) rank cur .. cur+g-1 (R19) become children prefix + j;
// lane t < g owns child t.  Child completion times C'_0 = C_0 + p_j0, C'_k = max(C'_k-1, C_k) + p_jk
// come from one serial pass over the machines per lane.
// A parent with children left is copied to the kept buffer, cursor advanced.
// Rows are 16-byte aligned (stride is a multiple of 8): copies move uint4s.
__global__ void expand_kernel(Nodes st, int64_t first, int64_t B, const int64_t *__restrict__ off,
                              Nodes ch, unsigned long long *ch_key, uint16_t *ch_uf, Nodes kp,
                              const int32_t *__restrict__ ptm, int n, int m, int stride, int by_idle,
                              uint16_t *ppf, int32_t *ch_par)
{
    extern __shared__ unsigned long long ex_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = (n + 31) >> 5;
    // per warp: keys[n] u64 | bm[nw] u32 | parent C[m] int32 (cs)
    unsigned long long *keys = ex_smem + (size_t)wib * (n + (nw + 1) / 2 + 16);
    uint32_t *bm = reinterpret_cast<uint32_t *>(keys + n);
    int32_t *cs = reinterpret_cast<int32_t *>(keys + n + (nw + 1) / 2);
    const int s8 = stride >> 3; // uint4 per row
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; p < B; p += warps) {
        const int64_t src = first + p;
        const uint4 *row4 = reinterpret_cast<const uint4 *>(st.pf + (size_t)src * stride);
        const int d = st.dp[src], cur = st.cur[src];
        const long long o0 = off[p], o1 = off[p + 1];
        const int g = (int)((o1 & 0xffffffffll) - (o0 & 0xffffffffll));
        const int keep = (int)((o1 >> 32) - (o0 >> 32));
        const int64_t c0 = o0 & 0xffffffffll;
        const int d8 = (d + 7) >> 3; // uint4 holding prefix entries
        long long klast = -1;        // key of the last child generated now
        if (g > 0) {
            // scheduled-job bitmap from the prefix, eight ids per load
            for (int w = lane; w < nw; w += 32) bm[w] = 0;
            __syncwarp();
            for (int q = lane; q < d8; q += 32) {
                const uint4 v = row4[q];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const uint32_t j = (t & 1) ? (w4[t >> 1] >> 16) : (w4[t >> 1] & 0xffffu);
                    if (q * 8 + t < d) atomicOr(&bm[j >> 5], 1u << (j & 31));
                }
            }
            __syncwarp();
            // candidates: the unscheduled jobs, compacted in j order into
            // keys[0..nc), then keyed (idle << 12) | j, lane per candidate, by
            // the idle time appending each opens on the machines (R19):
            // machine k, free at C_k, waits until j leaves machine k-1
            for (int k = lane; k < m; k += 32) cs[k] = st.C[(size_t)src * m + k];
            int nc = 0;
            for (int w = 0; w < nw; ++w) {
                const int j = w * 32 + lane;
                const bool cand = j < n && !(bm[w] >> lane & 1);
                const unsigned bal = __ballot_sync(0xffffffffu, cand);
                if (cand) keys[nc + __popc(bal & ((1u << lane) - 1))] = (unsigned long long)j;
                nc += __popc(bal);
            }
            __syncwarp();
            const bool v4 = (m & 3) == 0 && (reinterpret_cast<uintptr_t>(ptm) & 15) == 0;
            for (int i = lane; i < nc; i += 32) {
                const int j = (int)keys[i];
                long long idle = 0;
                int prev = 0;
                const int32_t *pj = ptm + (size_t)j * m;
                if (v4 && by_idle) { // 16-byte PTM loads (m % 4 == 0)
                    for (int k = 0; k < m; k += 4) {
                        const int4 pv = __ldg(reinterpret_cast<const int4 *>(pj + k));
                        const int pk[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int ck = cs[k + t];
                            const int start = max(ck, prev);
                            idle += start - ck;
                            prev = start + pk[t];
                        }
                    }
                } else {
#pragma unroll 4
                    for (int k = 0; k < (by_idle ? m : 0); ++k) { // (by_idle = 0: job order, A/B only)
                        const int ck = cs[k];
                        const int start = max(ck, prev);
                        idle += start - ck;
                        prev = start + __ldg(pj + k);
                    }
                }
                keys[i] = ((unsigned long long)idle << 12) | (unsigned)j;
            }
            __syncwarp();
            // children of this pop: the g smallest keys above the last key taken
            // (= key ranks cur .. cur+g-1), one warp-min round per child
            long long thr = st.kl[src];
            unsigned long long mykey = 0ull;
            // at most 32 candidates whose keys fit 32 bits (deep parents, the
            // bulk of the search): one bitonic sort of the warp's keys, then
            // the g keys after the ones already taken (<= thr) by shuffles
            bool sorted = false;
            if (nc <= 32) {
                const unsigned long long kk = lane < nc ? keys[lane] : 0ull;
                if (__all_sync(0xffffffffu, kk < 0xffffffffull)) {
                    uint32_t k32 = lane < nc ? (uint32_t)kk : 0xffffffffu;
#pragma unroll
                    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
                        for (int j = k >> 1; j > 0; j >>= 1) {
                            const uint32_t o = __shfl_xor_sync(0xffffffffu, k32, j);
                            const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
                            k32 = keep_min ? min(k32, o) : max(k32, o);
                        }
                    }
                    const int pos = __popc(__ballot_sync(0xffffffffu, lane < nc && (long long)k32 <= thr));
                    const uint32_t mine = __shfl_sync(0xffffffffu, k32, (pos + lane) & 31);
                    if (lane < g) mykey = mine;
                    if (g > 0) thr = (long long)__shfl_sync(0xffffffffu, k32, (pos + g - 1) & 31);
                    sorted = true;
                }
            }
            for (int t = 0; t < (sorted ? 0 : g); ++t) {
                unsigned long long best = ~0ull;
                for (int i = lane; i < nc; i += 32) {
                    const unsigned long long k = keys[i];
                    if ((long long)k > thr && k < best) best = k;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
                    best = y < best ? y : best;
                }
                if (lane == t) mykey = best;
                thr = (long long)best;
            }
            klast = thr;
            const int myj = lane < g ? (int)(mykey & 0xfffu) : -1;
            // each child's unscheduled jobs (the bounding kernel's input: n' - 1
            // entries instead of a d + 1 prefix): the parent's candidates, in
            // job order, without the child's own job
            if (ch_uf) {
                const unsigned lt = (1u << lane) - 1u;
                for (int t = 0; t < g; ++t) {
                    const int xj = __shfl_sync(0xffffffffu, myj, t);
                    uint16_t *ur = ch_uf + (size_t)(c0 + t) * stride;
                    int base = 0;
                    for (int i0 = 0; i0 < nc; i0 += 32) {
                        const int i = i0 + lane;
                        const int j = i < nc ? (int)(keys[i] & 0xfffu) : -1;
                        const bool keep = i < nc && j != xj;
                        const unsigned bal = __ballot_sync(0xffffffffu, keep);
                        if (keep) ur[base + __popc(bal & lt)] = (uint16_t)j;
                        base += __popc(bal);
                    }
                }
            }
            __syncwarp(); // keys are rewritten by the warp's next parent
            if (ppf) {
                // lazy rows: keep the parent's row once; a child's row (parent +
                // its job) is built only if it survives (scatter) or is the best
                // leaf (commit) — most children are pruned right after bounding
                uint4 *prow4 = reinterpret_cast<uint4 *>(ppf + (size_t)p * stride);
                for (int q = lane; q < d8; q += 32) prow4[q] = row4[q];
                if (lane < g) ch_par[c0 + lane] = (int32_t)p;
            } else {
                // prefixes: every child row = the parent's row with its job at d
                for (int t = 0; t < g; ++t) {
                    const int j = __shfl_sync(0xffffffffu, myj, t);
                    uint4 *crow4 = reinterpret_cast<uint4 *>(ch.pf + (size_t)(c0 + t) * stride);
                    for (int q = lane; q <= (d >> 3) && q < s8; q += 32) crow4[q] = child_vec(row4, d, j, q);
                }
            }
            // completion times, lane t for child t: C'_0 = C_0 + p_j0,
            // C'_k = max(C'_k-1, C_k) + p_jk, a serial max-plus pass over the
            // machines per lane (all g children at once)
            if (lane < g) {
                const int32_t *pj = ptm + (size_t)myj * m;
                int32_t *cc = ch.C + (size_t)(c0 + lane) * m;
                int prev = 0;
                if ((m & 3) == 0 && ((reinterpret_cast<uintptr_t>(cc) | reinterpret_cast<uintptr_t>(pj)) & 15) == 0) {
                    // 16-byte loads and stores; the parent's C from shared memory
                    for (int k = 0; k < m; k += 4) {
                        const int4 pv = __ldg(reinterpret_cast<const int4 *>(pj + k));
                        int4 o;
                        o.x = prev = max(prev, cs[k]) + pv.x;
                        o.y = prev = max(prev, cs[k + 1]) + pv.y;
                        o.z = prev = max(prev, cs[k + 2]) + pv.z;
                        o.w = prev = max(prev, cs[k + 3]) + pv.w;
                        *reinterpret_cast<int4 *>(cc + k) = o;
                    }
                } else {
#pragma unroll 4
                    for (int k = 0; k < m; ++k) {
                        prev = max(prev, cs[k]) + pj[k];
                        cc[k] = prev;
                    }
                }
                ch.dp[c0 + lane] = d + 1;
                ch_key[c0 + lane] = mykey;
            }
        }
        if (keep) {
            const int64_t dst = o0 >> 32;
            uint4 *krow4 = reinterpret_cast<uint4 *>(kp.pf + (size_t)dst * stride);
            for (int q = lane; q < d8; q += 32) krow4[q] = row4[q];
            for (int k = lane; k < m; k += 32) kp.C[(size_t)dst * m + k] = st.C[(size_t)src * m + k];
            if (lane == 0) {
                kp.dp[dst] = d;
                kp.cur[dst] = cur + g;
                kp.kl[dst] = klast;
                kp.lb[dst] = st.lb[src];
            }
        }
        __syncwarp();
    }
}

// Kept parents back onto the stack at [first, first + kept).
__global__ void restore_kernel(Nodes kp, const int64_t *off_B, int64_t first, Nodes st, int m,
                               int stride)
{
    const int64_t Pk = *off_B >> 32;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < Pk;
         q += warps) {
        const int d = kp.dp[q];
        const int64_t dst = first + q;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(kp.pf + (size_t)q * stride);
        uint4 *d4 = reinterpret_cast<uint4 *>(st.pf + (size_t)dst * stride);
        for (int i = lane; i < ((d + 7) >> 3); i += 32) d4[i] = s4[i];
        for (int k = lane; k < m; k += 32) st.C[(size_t)dst * m + k] = kp.C[(size_t)q * m + k];
        if (lane == 0) {
            st.dp[dst] = d;
            st.cur[dst] = kp.cur[q];
            st.kl[dst] = kp.kl[q];
            st.lb[dst] = kp.lb[q];
        }
    }
}

// Best-first among siblings (R10, R19): one warp per parent; its g children
// [c0, c0+g) get slots in descending (LB, key) order, so after compaction the
// best child is the top of the stack and is popped first.
__global__ void order_kernel(const int32_t *__restrict__ lb, const unsigned long long *__restrict__ key,
                             int64_t B, const int64_t *__restrict__ off, int32_t *ord)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < B; p += warps) {
        const int64_t c0 = off[p] & 0xffffffffll;
        const int g = (int)((off[p + 1] & 0xffffffffll) - c0);
        if (g == 0) continue;
        const int mylb = lane < g ? lb[c0 + lane] : 0;
        const unsigned long long myk = lane < g ? key[c0 + lane] : 0ull;
        int r = 0;
        for (int t = 0; t < g; ++t) {
            const int l = __shfl_sync(0xffffffffu, mylb, t);
            const unsigned long long k = __shfl_sync(0xffffffffu, myk, t);
            r += (l > mylb) || (l == mylb && k > myk);
        }
        if (lane < g) ord[c0 + r] = (int32_t)(c0 + lane);
    }
}

__global__ void iota_kernel(int32_t *ord, int64_t cnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) ord[i] = (int32_t)i;
}

// Elimination (a6) + leaves (a8): count survivors per block.
__global__ void __launch_bounds__(kPruneThreads)
    prune_kernel(Nodes ch, const int32_t *__restrict__ ord, const int64_t *count, int n, int m,
                 const int32_t *inc_dev, unsigned long long *cand, int32_t *bcnt,
                 unsigned long long *stats)
{
    const int64_t C = *count;
    // the grid covers the child buffer's capacity; blocks past this
    // iteration's children only report an empty count
    if ((int64_t)blockIdx.x * blockDim.x >= C) {
        if (threadIdx.x == 0) bcnt[blockIdx.x] = 0;
        return;
    }
    const int inc = *inc_dev;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int survive = 0, pruned = 0, leaf = 0;
    unsigned long long w = 0; // Fig. 3 / Table I operations of this child's bound (§7)
    if (i < C) {
        const int32_t rec = ord[i];
        const int d = ch.dp[rec], lb = ch.lb[rec];
        const unsigned long long P = (unsigned long long)m * (m - 1) / 2, np = (unsigned)(n - d);
        w = 2ull * d * m + np * (3ull * m - 2) + np * m + P * n + 4ull * P * np + 2ull * P;
        if (d >= n - 1) { // complete or forced completion: LB is its makespan (R6, P4)
            leaf = 1;
            if (lb < inc) atomicMin(cand, ((unsigned long long)(unsigned)lb << 32) | (unsigned)rec);
        } else if (lb < inc) {
            survive = 1;
        } else {
            pruned = 1;
        }
    }
    const int cs = __syncthreads_count(survive);
    const int cp = __syncthreads_count(pruned);
    const int cl = __syncthreads_count(leaf);
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(&stats[2], w);
    if (threadIdx.x == 0) {
        bcnt[blockIdx.x] = cs;
        if (cp) atomicAdd(&stats[0], (unsigned long long)cp);
        if (cl) atomicAdd(&stats[1], (unsigned long long)cl);
    }
}

// Stream compaction of the survivors onto the stack above the kept parents.
__global__ void __launch_bounds__(kPruneThreads)
    scatter_kernel(Nodes ch, const int32_t *__restrict__ ord, const int64_t *count,
                   const int64_t *off_B, int n, int m, int stride, const int32_t *inc_dev,
                   const int64_t *__restrict__ boff, int64_t first, Nodes st,
                   const uint16_t *__restrict__ ppf, const int32_t *__restrict__ ch_par,
                   const unsigned long long *__restrict__ ch_key)
{
    __shared__ int64_t s_dst[kPruneThreads];
    __shared__ int64_t s_src[kPruneThreads];
    const int64_t C = *count;
    if ((int64_t)blockIdx.x * blockDim.x >= C) return; // past this iteration's children
    const int64_t top = first + (*off_B >> 32);
    const int inc = *inc_dev;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int survive = 0;
    const int32_t rec = i < C ? ord[i] : 0;
    if (i < C) survive = ch.dp[rec] < n - 1 && ch.lb[rec] < inc;
    long long tot;
    const long long r = block_excl_scan(survive, tot);
    if (survive) {
        const int64_t dst = top + boff[blockIdx.x] + r;
        s_dst[r] = dst;
        s_src[r] = rec;
        st.dp[dst] = ch.dp[rec];
        st.cur[dst] = 0;
        st.kl[dst] = -1;
        st.lb[dst] = ch.lb[rec];
    }
    __syncthreads();
    // warp-cooperative, coalesced row copies; rows are 16-byte aligned (stride
    // is a multiple of 8), so prefixes move as uint4s (eight job ids each)
    // Four rows per warp in flight (loads of all four before their stores: the
    // copy is latency-bound, one row per warp left most of HBM idle).
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    constexpr int RU = 4;
    for (int k0 = wib; k0 < tot; k0 += RU * nwb) {
        int64_t src[RU], dst[RU];
        int d8[RU];
        uint4 v[RU];
        int cv[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int k = k0 + u * nwb;
            d8[u] = 0;
            if (k < tot) {
                src[u] = s_src[k];
                dst[u] = s_dst[k];
                const int dc = ch.dp[src[u]];
                d8[u] = (dc + 7) >> 3;
                if (lane < d8[u])
                    v[u] = ppf ? child_vec(reinterpret_cast<const uint4 *>(ppf + (size_t)ch_par[src[u]] * stride),
                                           dc - 1, (int)(ch_key[src[u]] & 0xfffu), lane)
                               : reinterpret_cast<const uint4 *>(ch.pf + (size_t)src[u] * stride)[lane];
                if (lane < m) cv[u] = ch.C[(size_t)src[u] * m + lane];
            }
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            if (k0 + u * nwb >= tot) continue;
            uint4 *drow = reinterpret_cast<uint4 *>(st.pf + (size_t)dst[u] * stride);
            const uint4 *srow = reinterpret_cast<const uint4 *>(ch.pf + (size_t)src[u] * stride);
            if (lane < d8[u]) drow[lane] = v[u];
            for (int q = lane + 32; q < d8[u]; q += 32) // rows beyond 256 jobs
                drow[q] = ppf ? child_vec(reinterpret_cast<const uint4 *>(ppf + (size_t)ch_par[src[u]] * stride),
                                          ch.dp[src[u]] - 1, (int)(ch_key[src[u]] & 0xfffu), q)
                              : srow[q];
            if (lane < m) st.C[(size_t)dst[u] * m + lane] = cv[u];
            for (int q = lane + 32; q < m; q += 32) st.C[(size_t)dst[u] * m + q] = ch.C[(size_t)src[u] * m + q];
        }
    }
}

// Adopt the best leaf of this iteration (a8) and publish the status.
__global__ void commit_kernel(Nodes ch, int n, int stride, int32_t *inc, unsigned long long *cand,
                              int32_t *perm, long long *packed, int rank, const int64_t *off_B,
                              const int64_t *T_dev, BBStatus *status, const uint16_t *ppf,
                              const int32_t *ch_par, const unsigned long long *ch_key)
{
    __shared__ int s_improved;
    __shared__ uint32_t s_bm[FSP_MAX_JOBS / 32];
    const unsigned long long c = *cand;
    if (threadIdx.x == 0) s_improved = 0;
    __syncthreads();
    if (c != kNoCand) {
        const int mk = (int)(c >> 32);
        const int64_t idx = (int64_t)(c & 0xffffffffull);
        if (mk < *inc) {
            // the leaf's row: its own, or (lazy rows) its parent's + its job
            const uint16_t *row = ppf ? ppf + (size_t)ch_par[idx] * stride : ch.pf + (size_t)idx * stride;
            const int d = ch.dp[idx];
            for (int w = threadIdx.x; w < (n + 31) / 32; w += blockDim.x) s_bm[w] = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < d; i += blockDim.x) {
                const int j = ppf && i == d - 1 ? (int)(ch_key[idx] & 0xfffu) : row[i];
                perm[i] = j;
                atomicOr(&s_bm[j >> 5], 1u << (j & 31));
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                if (d == n - 1) // the forced completion: the one job left
                    for (int j = 0; j < n; ++j)
                        if (!(s_bm[j >> 5] >> (j & 31) & 1)) perm[n - 1] = j;
                *inc = mk;
                s_improved = 1;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *cand = kNoCand;
        // (own best << 32) | rank: the MIN over ranks names the holder of the
        // best permutation (an adopted incumbent only tightens pruning)
        if (s_improved) *packed = ((long long)*inc << 32) | (unsigned)rank;
        status->children = *off_B & 0xffffffffll;
        status->kept = *off_B >> 32;
        status->survivors = *T_dev;
        status->incumbent = *inc;
        status->improved = s_improved;
    }
}

__global__ void adopt_ub_kernel(int32_t *inc, const long long *src)
{
    const int g = (int)(*src >> 32);
    if (g < *inc) *inc = g;
}

int cuda_or(cudaError_t e, const char *what) { return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, what); }

void free_nodes(Nodes &x)
{
    cudaFree(x.pf);
    cudaFree(x.dp);
    cudaFree(x.C);
    cudaFree(x.cur);
    cudaFree(x.lb);
    cudaFree(x.kl);
    x = Nodes();
}

void bb_free(BBState *s)
{
    if (!s) return;
    free_nodes(s->st);
    free_nodes(s->kp);
    free_nodes(s->ch);
    cudaFree(s->ch_key);
    cudaFree(s->ch_uf);
    cudaFree(s->ppf);
    cudaFree(s->ch_par);
    cudaFree(s->ord);
    cudaFree(s->d_maxnp);
    cudaFree(s->d_famflag);
    cudaFree(s->d_count_sparse);
    cudaFree(s->plan);
    cudaFree(s->off);
    cudaFree(s->d_count);
    cudaFree(s->boff);
    cudaFree(s->bcnt);
    cudaFree(s->tsum);
    cudaFree(s->toff);
    cudaFree(s->d_inc);
    cudaFree(s->d_cand);
    cudaFree(s->d_packed);
    cudaFree(s->d_scratch);
    cudaFree(s->d_perm);
    cudaFree(s->d_stats);
    cudaFree(s->d_status);
    if (s->h_status) cudaFreeHost(s->h_status);
    if (s->ev_in) cudaEventDestroy(s->ev_in);
    if (s->ev_out) cudaEventDestroy(s->ev_out);
    if (s->ev_t0) cudaEventDestroy(s->ev_t0);
    if (s->ev_t1) cudaEventDestroy(s->ev_t1);
    if (s->timing)
        fprintf(stderr, "FSP_BB_TIMING: %lld iterations, device time %.3f s\n", (long long)s->stats.iterations,
                s->gpu_ms / 1e3);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

int64_t env_i64(const char *name, int64_t dflt)
{
    const char *v = getenv(name);
    return v ? atoll(v) : dflt;
}

size_t node_bytes(const BBState *s) { return (size_t)s->stride * 2 + 20 + (size_t)s->m * 4; }

cudaError_t alloc_nodes(Nodes &x, int64_t cnt, int stride, int m)
{
    cudaError_t e = cudaMalloc(&x.pf, (size_t)cnt * stride * 2);
    if (e == cudaSuccess) e = cudaMalloc(&x.dp, (size_t)cnt * 4);
    if (e == cudaSuccess) e = cudaMalloc(&x.C, (size_t)cnt * m * 4);
    if (e == cudaSuccess) e = cudaMalloc(&x.cur, (size_t)cnt * 4);
    if (e == cudaSuccess) e = cudaMalloc(&x.lb, (size_t)cnt * 4);
    if (e == cudaSuccess) e = cudaMalloc(&x.kl, (size_t)cnt * 8);
    return e;
}

// Copy k nodes between node arrays (device to device, stream-ordered).
cudaError_t copy_nodes(const BBState *s, Nodes dst, int64_t di, Nodes src, int64_t si, int64_t k)
{
    const int st = s->stride, m = s->m;
    cudaStream_t q = s->stream;
    cudaError_t e = cudaMemcpyAsync(dst.pf + (size_t)di * st, src.pf + (size_t)si * st,
                                    (size_t)k * st * 2, cudaMemcpyDeviceToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dst.dp + di, src.dp + si, (size_t)k * 4, cudaMemcpyDeviceToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dst.C + (size_t)di * m, src.C + (size_t)si * m, (size_t)k * m * 4,
                            cudaMemcpyDeviceToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dst.cur + di, src.cur + si, (size_t)k * 4, cudaMemcpyDeviceToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dst.lb + di, src.lb + si, (size_t)k * 4, cudaMemcpyDeviceToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(dst.kl + di, src.kl + si, (size_t)k * 8, cudaMemcpyDeviceToDevice, q);
    return e;
}

// A flat buffer of k nodes viewed as node arrays:
// [k] last-key i64 | [k][stride] u16 prefixes | [k] depth | [k][m] C | [k] cursor | [k] LB.
Nodes flat_view(const BBState *s, const void *buf, int64_t k)
{
    uint8_t *b = static_cast<uint8_t *>(const_cast<void *>(buf));
    Nodes x;
    x.kl = reinterpret_cast<long long *>(b);
    b += (size_t)k * 8;
    x.pf = reinterpret_cast<uint16_t *>(b);
    b += (size_t)k * s->stride * 2;
    x.dp = reinterpret_cast<int32_t *>(b);
    b += (size_t)k * 4;
    x.C = reinterpret_cast<int32_t *>(b);
    b += (size_t)k * s->m * 4;
    x.cur = reinterpret_cast<int32_t *>(b);
    b += (size_t)k * 4;
    x.lb = reinterpret_cast<int32_t *>(b);
    return x;
}

// Push nodes given as (depth, prefix) host rows onto the stack top; their
// completion times are computed here from the prefixes.
int push_host(BBState *s, const std::vector<uint16_t> &pf, const std::vector<int32_t> &dp)
{
    const int64_t k = (int64_t)dp.size();
    if (s->size + k > s->cap) return fsp_fail(FSP_ENOMEM, "B&B stack full");
    const int m = s->m;
    const int32_t *ptm = s->inst->h_ptm;
    std::vector<int32_t> C((size_t)k * m, 0), zero((size_t)k, 0);
    for (int64_t i = 0; i < k; ++i) {
        int32_t *c = &C[(size_t)i * m];
        for (int q = 0; q < dp[i]; ++q) {
            const int j = pf[(size_t)i * s->stride + q];
            int prev = 0;
            for (int t = 0; t < m; ++t) {
                prev = std::max(prev, c[t]) + ptm[(size_t)j * m + t];
                c[t] = prev;
            }
        }
    }
    const int64_t at = s->size;
    cudaStream_t q = s->stream;
    cudaError_t e = cudaMemcpyAsync(s->st.pf + (size_t)at * s->stride, pf.data(),
                                    sizeof(uint16_t) * pf.size(), cudaMemcpyHostToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->st.dp + at, dp.data(), 4 * k, cudaMemcpyHostToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->st.C + (size_t)at * m, C.data(), 4 * C.size(), cudaMemcpyHostToDevice, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->st.cur + at, zero.data(), 4 * k, cudaMemcpyHostToDevice, q);
    if (e == cudaSuccess) // never bounded: LB 0, never eliminated at pop
        e = cudaMemcpyAsync(s->st.lb + at, zero.data(), 4 * k, cudaMemcpyHostToDevice, q);
    std::vector<long long> none((size_t)k, -1);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->st.kl + at, none.data(), 8 * k, cudaMemcpyHostToDevice, q);
    if (e == cudaSuccess) e = cudaStreamSynchronize(q);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B push");
    s->size += k;
    return FSP_OK;
}

void device_scan(BBState *s, const long long *in64, const int32_t *in32, int64_t N, int64_t *out,
                 int64_t *count_out)
{
    cudaStream_t st = s->stream;
    if (N <= 4 * kScanThreads) {
        scan_kernel<<<1, kScanThreads, 0, st>>>(in64, in32, N, out, count_out);
        return;
    }
    const int64_t tiles = (N + kScanThreads - 1) / kScanThreads;
    scan_local_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(in64, in32, N, out, s->tsum);
    scan_kernel<<<1, kScanThreads, 0, st>>>(s->tsum, nullptr, tiles, s->toff, nullptr);
    scan_add_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(N, out, s->toff);
    scan_total_kernel<<<1, 1, 0, st>>>(N, out, s->toff, tiles, count_out);
}

// One select / branch / bound / eliminate iteration.
int bb_iterate(BBState *s)
{
    const fsp_instance *inst = s->inst;
    const int n = s->n, m = s->m, stride = s->stride;
    cudaStream_t st = s->stream;
    const int64_t open = s->size - s->base;
    if (open <= 0) return FSP_OK;
    // the first dive (a9): one parent per iteration, all its children (up to
    // 32, best idle first) bounded and ordered, for the first dive_iters
    // iterations: a depth-first descent along the best child that sets the
    // first incumbent (SURVEY.md §8(d) C4 "first dive sets it"); then batches
    const bool dive = s->stats.iterations < s->dive_iters;
    const int K = dive ? 32 : s->K;
    if (s->timing) cudaEventRecord(s->ev_t0, st);
    // B parents: at most K children each fit the child buffer; the stack grows
    // by at most B*K per iteration and B*K*n over a descent, held under half
    // the capacity (the beam); n*K slots of headroom are always left
    const int64_t usable = s->cap - (int64_t)n * K;
    int64_t B = std::min<int64_t>(open, std::min<int64_t>(s->kcap, s->ccap / K));
    B = std::min<int64_t>(B, std::max<int64_t>(1, (int64_t)(s->cap * s->beam) / ((int64_t)K * n)));
    B = std::min<int64_t>(B, std::max<int64_t>(1, (usable - s->size) / K));
    if (dive) B = 1;
    if (s->size + B * K > s->cap) return fsp_fail(FSP_ENOMEM, "B&B stack full");
    const int64_t first = s->size - B;

    const int pb = 256;
    if (s->family) {
        cudaError_t e0 = cudaMemsetAsync(s->d_maxnp, 0, 4, st);
        if (e0 != cudaSuccess) return fsp_cuda_fail(e0, "B&B iteration");
    }
    plan_kernel<<<(unsigned)((B + pb - 1) / pb), pb, 0, st>>>(s->st, first, B, n, K, s->d_inc, s->plan,
                                                              s->d_stats, s->d_maxnp);
    device_scan(s, s->plan, nullptr, B, s->off, s->d_count);
    if (s->family)
        route_kernel<<<1, 1, 0, st>>>(s->d_maxnp, s->d_count, 1, s->d_famflag, s->d_count_sparse);
    const int ewarps = n > 1024 ? 1 : 4;
    const int eblocks = (int)std::min<int64_t>((B + ewarps - 1) / ewarps, 148 * 32);
    const size_t esmem = (size_t)ewarps * 8 * (n + ((n + 31) / 32 + 1) / 2 + 16);
    expand_kernel<<<eblocks, ewarps * 32, esmem, st>>>(s->st, first, B, s->off, s->ch, s->ch_key,
                                                       s->ch_uf, s->kp, inst->d_ptm32, n, m, stride,
                                                       s->order, s->ppf, s->ch_par);
    const int64_t *off_B = s->off + B; // (kept << 32) | children, on the device
    // bounding (before the kept parents overwrite the popped range): the
    // family kernel from the parents (one of the two launches exits at once),
    // or the lb kernel with the sparse-walk plan, pool size read on the device
    // (the lb kernel first: a couple-split launch clears lb_out before it runs)
    const int64_t maxC = B * K;
    int rc = fsp_launch_lb_dev(inst, s->ch.pf, stride, s->ch.dp, maxC,
                               s->family ? s->d_count_sparse : s->d_count, s->ch.C, m, s->sparse, s->ch.lb,
                               st, 0, s->ch_uf);
    if (rc != FSP_OK) return rc;
    if (s->family) {
        rc = fsp_launch_family(inst, s->st.pf + (size_t)first * stride, stride, s->st.dp + first,
                               s->st.C + (size_t)first * m, B, s->off, s->ch_key, s->ch.lb, s->d_famflag,
                               st);
        if (rc != FSP_OK) return rc;
    }
    restore_kernel<<<eblocks, ewarps * 32, 0, st>>>(s->kp, off_B, first, s->st, m, stride);
    if (s->order) {
        order_kernel<<<eblocks, ewarps * 32, 0, st>>>(s->ch.lb, s->ch_key, B, s->off, s->ord);
    } else { // (A/B: children in generation order)
        iota_kernel<<<(unsigned)((B * K + 255) / 256), 256, 0, st>>>(s->ord, B * K);
    }
    const int nblk = (int)((maxC + kPruneThreads - 1) / kPruneThreads);
    prune_kernel<<<nblk, kPruneThreads, 0, st>>>(s->ch, s->ord, s->d_count, n, m, s->d_inc, s->d_cand,
                                                  s->bcnt, s->d_stats);
    device_scan(s, nullptr, s->bcnt, nblk, s->boff, nullptr);
    scatter_kernel<<<nblk, kPruneThreads, 0, st>>>(s->ch, s->ord, s->d_count, off_B, n, m, stride,
                                                    s->d_inc, s->boff, first, s->st, s->ppf, s->ch_par,
                                                    s->ch_key);
    commit_kernel<<<1, 256, 0, st>>>(s->ch, n, stride, s->d_inc, s->d_cand, s->d_perm, s->d_packed,
                                     s->rank, off_B, s->boff + nblk, s->d_status, s->ppf, s->ch_par,
                                     s->ch_key);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && s->timing) e = cudaEventRecord(s->ev_t1, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->h_status, s->d_status, sizeof(BBStatus), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B iteration");
    if (s->timing) { // diagnostics (FSP_BB_TIMING): device time of the iteration's kernels
        float ms = 0;
        cudaEventElapsedTime(&ms, s->ev_t0, s->ev_t1);
        s->gpu_ms += ms;
    }
    s->size = first + s->h_status->kept + s->h_status->survivors;
    s->last_children = s->h_status->children;
    s->stats.bounded += s->h_status->children;
    s->stats.branched += B;
    s->stats.iterations += 1;
    if (s->h_status->improved) {
        s->have = 1;
        s->perm_ms = s->h_status->incumbent;
    }
    return FSP_OK;
}

int bb_create(const fsp_instance *inst, int32_t initial_ub, int32_t rank, int32_t world,
              void *stream, BBState **out, double mem_frac = 0.0, int64_t children_cap = 0,
              bool root_only = false)
{
    if (!inst || !out || world < 1 || rank < 0 || rank >= world || initial_ub < 0)
        return fsp_fail(FSP_EINVAL, "bad B&B arguments");
    BBState *s = new (std::nothrow) BBState();
    if (!s) return fsp_fail(FSP_ENOMEM, "host allocation");
    s->inst = inst;
    s->rank = rank;
    s->world = world;
    s->n = inst->n;
    s->m = inst->m;
    s->stride = (inst->n + 7) & ~7;
    s->initial_inc = initial_ub == INT32_MAX ? INT32_MAX : initial_ub + 1; // R9
    s->sparse = getenv("FSP_BB_SPARSE") ? atoi(getenv("FSP_BB_SPARSE")) != 0 : true;
    // children per parent per pop: one lane per child in expand/order, K <= 32
    s->K = (int)std::min<int64_t>(32, std::max<int64_t>(1, env_i64("FSP_BB_K", 12)));
    s->order = env_i64("FSP_BB_ORDER", 1) != 0 ? 1 : 0;
    // the beam: B*K*n <= beam * capacity.  A descent pushes at most B*K nodes
    // per level, and every iteration's B is also held to the free stack
    // (usable - size) / K, so a beam above 1 never overflows: near a full stack
    // the batches shrink.  Measured at 200x20 (profiles/r02/bb_beam.txt):
    // 0.5 -> 4.7e8 nodes/s, 2 -> 5.9e8, 4 -> 6.3e8 (30 s), 8 no further gain
    s->beam = getenv("FSP_BB_BEAM") ? atof(getenv("FSP_BB_BEAM")) : 4.0;
    s->dive_iters = s->order ? std::max<int64_t>(0, env_i64("FSP_BB_DIVE", s->n)) : 0;
    // sibling-incremental bounding (family.cu) for batches of parents with <= 32
    // unscheduled jobs: measured slower than the sparse walk at the B&B's
    // depth mix, so opt-in (FSP_BB_FAMILY=1)
    s->family = inst->fam.warps > 0 && env_i64("FSP_BB_FAMILY", 0) != 0;
    cudaError_t e = cudaSuccess;
    if (stream) {
        s->stream = static_cast<cudaStream_t>(stream);
    } else {
        e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        s->own_stream = true;
    }
    const int n = s->n, m = s->m;
    size_t freeb = 0, totalb = 0;
    if (e == cudaSuccess) e = cudaMemGetInfo(&freeb, &totalb);
    // children per iteration: enough to fill the GPU several times over
    s->ccap = std::max<int64_t>(children_cap > 0 ? children_cap : env_i64("FSP_BB_CHILDREN", 1 << 22), 32);
    s->kcap = s->ccap;
    // the stack takes most of the free HBM (180 GB per B200)
    const double frac = mem_frac > 0 ? mem_frac
                        : getenv("FSP_BB_MEM_FRAC") ? atof(getenv("FSP_BB_MEM_FRAC")) : 0.5;
    const size_t buffers = (size_t)(s->ccap + s->kcap) * node_bytes(s);
    int64_t cap = freeb > buffers ? (int64_t)((double)(freeb - buffers) * frac / node_bytes(s)) : 0;
    cap = env_i64("FSP_BB_STACK", std::min<int64_t>(cap, (int64_t)1 << 31));
    s->cap = std::max<int64_t>(cap, (int64_t)n * 32 * 4); // the dive pushes up to 32 per level
    const int64_t nblk = (s->ccap + kPruneThreads - 1) / kPruneThreads + 1;
    if (e == cudaSuccess) e = alloc_nodes(s->st, s->cap, s->stride, m);
    if (e == cudaSuccess) e = alloc_nodes(s->kp, s->kcap, s->stride, m);
    if (e == cudaSuccess) e = alloc_nodes(s->ch, s->ccap, s->stride, m);
    auto alloc = [&](void **p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(p, bytes);
    };
    alloc((void **)&s->ch_key, (size_t)s->ccap * 8);
    // unscheduled lists for the sparse byte-row bounding plan (long prefixes:
    // deep children have n' << d); measured slower for n < 64 (dense plan)
    if (env_i64("FSP_BB_ULIST", 1) != 0 && inst->plan_bb.sparse && inst->plan_bb.byte_rows) {
        alloc((void **)&s->ch_uf, (size_t)s->ccap * s->stride * 2);
        // the bounding then reads no child prefix: rows are built only for
        // the survivors and the best leaf (FSP_BB_LAZY=0: every child's row)
        if (env_i64("FSP_BB_LAZY", 1) != 0) {
            alloc((void **)&s->ppf, (size_t)s->kcap * s->stride * 2);
            alloc((void **)&s->ch_par, (size_t)s->ccap * 4);
        }
    }
    alloc((void **)&s->ord, (size_t)s->ccap * 4);
    alloc((void **)&s->d_maxnp, 4);
    alloc((void **)&s->d_famflag, 4);
    alloc((void **)&s->d_count_sparse, 8);
    alloc((void **)&s->plan, (size_t)s->kcap * 8);
    alloc((void **)&s->off, (size_t)(s->kcap + 1) * 8);
    alloc((void **)&s->d_count, 8);
    alloc((void **)&s->boff, (size_t)(nblk + 1) * 8);
    alloc((void **)&s->bcnt, (size_t)nblk * 4);
    alloc((void **)&s->tsum, (size_t)(s->kcap / kScanThreads + 2) * 8);
    alloc((void **)&s->toff, (size_t)(s->kcap / kScanThreads + 3) * 8);
    alloc((void **)&s->d_inc, 4);
    alloc((void **)&s->d_cand, 8);
    alloc((void **)&s->d_packed, 8);
    alloc((void **)&s->d_scratch, 8);
    alloc((void **)&s->d_perm, (size_t)n * 4);
    alloc((void **)&s->d_stats, 24);
    alloc((void **)&s->d_status, sizeof(BBStatus));
    if (e == cudaSuccess) e = cudaMallocHost((void **)&s->h_status, sizeof(BBStatus));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_out, cudaEventDisableTiming);
    s->timing = env_i64("FSP_BB_TIMING", 0) != 0;
    if (e == cudaSuccess && s->timing) e = cudaEventCreate(&s->ev_t0);
    if (e == cudaSuccess && s->timing) e = cudaEventCreate(&s->ev_t1);
    if (e == cudaSuccess) e = cudaMemcpy(s->d_inc, &s->initial_inc, 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(s->d_cand, 0xff, 8);
    if (e == cudaSuccess) e = cudaMemset(s->d_stats, 0, 24);
    if (e == cudaSuccess) {
        const long long pk = ((long long)INT32_MAX << 32) | (unsigned)rank; // no schedule yet
        e = cudaMemcpy(s->d_packed, &pk, 8, cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        bb_free(s);
        return fsp_cuda_fail(e, "B&B allocation");
    }
    // initial split: one rank keeps the root; with several ranks, rank r keeps
    // the depth-1 nodes j with j % world == r
    std::vector<uint16_t> pf;
    std::vector<int32_t> dp;
    if (world == 1 || n == 1 || root_only) {
        // (n == 1: the one depth-1 node is a complete schedule, which is only
        // evaluated as a child; root_only: the other ranks get work by
        // stealing; in both, rank 0 starts from the root, the others empty)
        if (rank == 0) {
            pf.assign(s->stride, 0xffff);
            dp.push_back(0);
        }
    } else {
        for (int j = n - 1; j >= 0; --j) {
            if (j % world != rank) continue;
            std::vector<uint16_t> row(s->stride, 0xffff);
            row[0] = (uint16_t)j;
            pf.insert(pf.end(), row.begin(), row.end());
            dp.push_back(1);
        }
    }
    int rc = dp.empty() ? FSP_OK : push_host(s, pf, dp);
    if (rc != FSP_OK) {
        bb_free(s);
        return rc;
    }
    *out = s;
    return FSP_OK;
}

int read_stats(BBState *s)
{
    unsigned long long h[3] = {0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(h, s->d_stats, 24, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B stats");
    s->stats.pruned = (int64_t)h[0];
    s->stats.leaves = (int64_t)h[1];
    s->stats.lb_ops = (int64_t)h[2];
    return FSP_OK;
}

int result(BBState *s, int32_t *makespan_out, int32_t *perm_out)
{
    cudaError_t e = cudaSuccess;
    if (perm_out && s->have)
        e = cudaMemcpyAsync(perm_out, s->d_perm, sizeof(int32_t) * s->n, cudaMemcpyDeviceToHost,
                            s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B result");
    if (makespan_out) *makespan_out = s->have ? s->perm_ms : -1;
    return s->have ? FSP_OK : fsp_fail(FSP_ENOTFOUND, "no schedule within the upper bound");
}

} // namespace

extern "C" int fsp_bb_solve(const fsp_instance *inst, int32_t initial_ub, int64_t max_nodes,
                            double time_limit_s, int32_t *makespan_out, int32_t *perm_out,
                            fsp_bb_stats *stats)
{
    if (!inst || !makespan_out || !perm_out) return fsp_fail(FSP_EINVAL, "null pointer");
    const auto t0 = std::chrono::steady_clock::now();
    BBState *s = nullptr;
    int rc = bb_create(inst, initial_ub, 0, 1, nullptr, &s);
    if (rc != FSP_OK) return rc;
    bool budget = false;
    while (s->size > s->base) {
        rc = bb_iterate(s);
        if (rc != FSP_OK) break;
        const double el =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if ((max_nodes > 0 && s->stats.bounded >= max_nodes) ||
            (time_limit_s > 0 && el >= time_limit_s)) {
            budget = s->size > s->base;
            break;
        }
    }
    if (rc == FSP_OK) rc = read_stats(s);
    s->stats.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats) *stats = s->stats;
    if (rc == FSP_OK) {
        rc = result(s, makespan_out, perm_out);
        if (budget) rc = fsp_fail(s->have ? FSP_EBUDGET : FSP_ENOTFOUND, "B&B budget exhausted");
    }
    bb_free(s);
    return rc;
}

// (hybrid.cu: several states on one device share its memory)
int fsp_bb_init_ex(const fsp_instance *inst, int32_t initial_ub, int32_t rank, int32_t world,
                   double mem_frac, int64_t children_cap, bool root_only, void **state)
{
    if (!state) return fsp_fail(FSP_EINVAL, "null state");
    BBState *s = nullptr;
    int rc = bb_create(inst, initial_ub, rank, world, nullptr, &s, mem_frac, children_cap, root_only);
    *state = s;
    return rc;
}

extern "C" int fsp_bb_init(const fsp_instance *inst, int32_t initial_ub, int32_t rank,
                           int32_t world, void **state)
{
    if (!state) return fsp_fail(FSP_EINVAL, "null state");
    BBState *s = nullptr;
    int rc = bb_create(inst, initial_ub, rank, world, nullptr, &s);
    *state = s;
    return rc;
}

extern "C" int fsp_bb_step(void *state, int32_t iters, void *cuda_stream)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || iters < 0) return fsp_fail(FSP_EINVAL, "bad B&B state");
    // the iterations run on the state's stream, ordered after the work already
    // queued on cuda_stream; later work on cuda_stream is ordered after them
    cudaStream_t cs = static_cast<cudaStream_t>(cuda_stream);
    cudaError_t e = cudaEventRecord(s->ev_in, cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, s->ev_in, 0);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B step ordering");
    int rc = FSP_OK;
    for (int i = 0; i < iters && s->size > s->base && rc == FSP_OK; ++i) rc = bb_iterate(s);
    if (rc == FSP_OK) rc = read_stats(s);
    e = cudaEventRecord(s->ev_out, s->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, s->ev_out, 0);
    if (e != cudaSuccess && rc == FSP_OK) rc = fsp_cuda_fail(e, "B&B step ordering");
    return rc;
}

// Test hook: the child pool of the last iteration (every child bounded, pruned
// or not), flat HOST layout [k][stride] u16 prefixes | [k] depth | [k][m] C |
// [k] LB, k = min(max_nodes, children of that iteration).
extern "C" int fsp_bb_debug_children(void *state, int64_t max_nodes, void *h_buf, int64_t *n_out)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !n_out || max_nodes < 0 || (max_nodes > 0 && !h_buf))
        return fsp_fail(FSP_EINVAL, "bad debug arguments");
    if (max_nodes == 0) { // query: children available
        *n_out = s->last_children;
        return FSP_OK;
    }
    const int64_t k = std::min(max_nodes, s->last_children);
    *n_out = k;
    if (k == 0) return FSP_OK;
    if (s->ppf) { // lazy rows: build the children's prefixes first
        materialize_kernel<<<(unsigned)std::min<int64_t>((k + 7) / 8, 148 * 16), 256, 0, s->stream>>>(
            s->ppf, s->ch_par, s->ch_key, s->ch.dp, k, s->stride, s->ch.pf);
        cudaError_t e0 = cudaGetLastError();
        if (e0 != cudaSuccess) return fsp_cuda_fail(e0, "debug children");
    }
    uint8_t *b = static_cast<uint8_t *>(h_buf);
    const size_t pfb = (size_t)k * s->stride * 2, cb = (size_t)k * s->m * 4;
    cudaStream_t q = s->stream;
    cudaError_t e = cudaMemcpyAsync(b, s->ch.pf, pfb, cudaMemcpyDeviceToHost, q);
    if (e == cudaSuccess) e = cudaMemcpyAsync(b + pfb, s->ch.dp, (size_t)k * 4, cudaMemcpyDeviceToHost, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(b + pfb + (size_t)k * 4, s->ch.C, cb, cudaMemcpyDeviceToHost, q);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(b + pfb + (size_t)k * 4 + cb, s->ch.lb, (size_t)k * 4,
                            cudaMemcpyDeviceToHost, q);
    if (e == cudaSuccess) e = cudaStreamSynchronize(q);
    return cuda_or(e, "debug children");
}

extern "C" int fsp_bb_ub_publish(void *state, int64_t *d_dst, void *stream)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !d_dst) return fsp_fail(FSP_EINVAL, "bad B&B state");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    // the packed word is current after every iteration (commit_kernel)
    cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_dst, s->d_packed, 8, cudaMemcpyDeviceToDevice, st);
    return cuda_or(e, "ub publish");
}

extern "C" int fsp_bb_ub_adopt(void *state, const int64_t *d_src, void *stream)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !d_src) return fsp_fail(FSP_EINVAL, "bad B&B state");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    adopt_ub_kernel<<<1, 1, 0, st>>>(s->d_inc, reinterpret_cast<const long long *>(d_src));
    return cuda_or(cudaStreamSynchronize(st), "ub adopt");
}

extern "C" int fsp_bb_ub_get(void *state, int64_t *packed)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !packed) return fsp_fail(FSP_EINVAL, "bad B&B state");
    cudaError_t e = cudaMemcpyAsync(packed, s->d_packed, 8, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    return cuda_or(e, "ub get");
}

extern "C" int fsp_bb_ub_set(void *state, int64_t packed)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s) return fsp_fail(FSP_EINVAL, "bad B&B state");
    cudaError_t e = cudaMemcpyAsync(s->d_scratch, &packed, 8, cudaMemcpyHostToDevice, s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "ub set");
    adopt_ub_kernel<<<1, 1, 0, s->stream>>>(s->d_inc, s->d_scratch);
    return cuda_or(cudaStreamSynchronize(s->stream), "ub set");
}

extern "C" int fsp_bb_pool_size(void *state, int64_t *n)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !n) return fsp_fail(FSP_EINVAL, "bad B&B state");
    *n = s->size - s->base;
    return FSP_OK;
}

extern "C" int64_t fsp_bb_node_bytes(void *state)
{
    BBState *s = static_cast<BBState *>(state);
    return s ? (int64_t)node_bytes(s) : 0;
}

// Donor side: the shallowest open nodes (bottom of the stack, the largest
// subtrees) go out as one flat buffer of fsp_bb_node_bytes per node:
// [k] last-key i64 | [k][stride] u16 prefixes | [k] depth | [k][m] C | [k] cursor | [k] LB.
extern "C" int fsp_bb_export(void *state, int64_t max_nodes, void *d_buf, int64_t *n_out)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !n_out || max_nodes < 0 || (max_nodes > 0 && !d_buf))
        return fsp_fail(FSP_EINVAL, "bad export arguments");
    const int64_t k = std::min(max_nodes, s->size - s->base);
    *n_out = k;
    if (k == 0) return FSP_OK;
    cudaError_t e = copy_nodes(s, flat_view(s, d_buf, k), 0, s->st, s->base, k);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "export");
    s->base += k;
    if (s->base == s->size) s->base = s->size = 0;
    return FSP_OK;
}

extern "C" int fsp_bb_import(void *state, const void *d_buf, int64_t k)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || k < 0 || (k > 0 && !d_buf)) return fsp_fail(FSP_EINVAL, "bad import arguments");
    if (k == 0) return FSP_OK;
    cudaError_t e = cudaSuccess;
    if (s->base > 0) { // compact the deque: move [base, size) down in non-overlapping chunks
        const int64_t open = s->size - s->base;
        for (int64_t q = 0; q < open && e == cudaSuccess; q += s->base)
            e = copy_nodes(s, s->st, q, s->st, s->base + q, std::min(s->base, open - q));
        if (e != cudaSuccess) return fsp_cuda_fail(e, "import compaction");
        s->size = open;
        s->base = 0;
    }
    if (s->size + k > s->cap) return fsp_fail(FSP_ENOMEM, "B&B stack full");
    e = copy_nodes(s, s->st, s->size, flat_view(s, d_buf, k), 0, k);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "import");
    s->size += k;
    return FSP_OK;
}

extern "C" int fsp_bb_result(void *state, int32_t *makespan_out, int32_t *perm_out)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s) return fsp_fail(FSP_EINVAL, "bad B&B state");
    return result(s, makespan_out, perm_out);
}

extern "C" int fsp_bb_get_stats(void *state, fsp_bb_stats *stats)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !stats) return fsp_fail(FSP_EINVAL, "bad B&B state");
    int rc = read_stats(s);
    *stats = s->stats;
    return rc;
}

extern "C" void fsp_bb_free(void *state) { bb_free(static_cast<BBState *>(state)); }
