// bb.cu — device-resident B&B for the permutation FSP.
//
// The four operators of §II-A with the paper's forward branching
// and elimination LB >= incumbent (R9), all on the device:
//   selection  (a9)  the top B open nodes of a device stack: deepest-first
//                    batches replace the paper's host best-first list (R10);
//   branching  (a7)  expand_kernel writes every child prefix + j, j unscheduled,
//                    ascending j;
//   bounding   (a1-a5) the LB kernel of lb_kernel.cu on the child pool, pool
//                    size read on the device;
//   elimination (a6) prune_kernel + scan + scatter_kernel: survivors LB <
//                    incumbent are stream-compacted back onto the stack in
//                    child order; leaves (depth >= n-1, whose LB is their exact
//                    makespan, R6) feed a packed (makespan, index) atomicMin and
//                    commit_kernel adopts the best one with its permutation (a8).
// One 24-byte status read per iteration is the only host round trip.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
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
    long long survivors; // pushed back onto the stack
    int incumbent;       // current incumbent (INT_MAX = none)
    int improved;        // incumbent improved this iteration
};

struct BBState {
    const fsp_instance *inst;
    int rank, world, n, stride;
    int64_t cap;         // stack capacity (nodes)
    int64_t base, size;  // open nodes live in [base, size)
    int64_t ccap;        // child buffer capacity
    uint16_t *st_pf;     // stack prefixes [cap][stride]
    int32_t *st_dp;      // stack depths
    uint16_t *ch_pf;     // children [ccap][stride]
    int32_t *ch_dp, *ch_lb;
    int64_t *off;        // children offsets per parent [ccap/1 + 1]
    int64_t *boff;       // survivor offsets per prune block
    int32_t *bcnt;       // survivor count per prune block
    int32_t *d_inc;      // incumbent makespan
    unsigned long long *d_cand;
    long long *d_packed; // (incumbent << 32) | rank for the MIN all-reduce
    long long *d_scratch;
    int32_t *d_perm;     // incumbent permutation
    unsigned long long *d_stats; // [pruned, leaves]
    BBStatus *d_status;
    BBStatus *h_status;  // pinned
    cudaStream_t stream;
    bool own_stream;
    fsp_bb_stats stats;
    int have;            // this rank holds a permutation ...
    int32_t perm_ms;     // ... of this makespan (the incumbent may be lower: adopted)
    double kids_per_parent; // running estimate for the batch size
    int32_t initial_inc; // initial_ub + 1 (saturating)
};

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int &total)
{
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// Block-wide exclusive scan of one int per thread (blockDim multiple of 32).
__device__ __forceinline__ long long block_excl_scan(int v, long long &total)
{
    __shared__ int wsum[32];
    __shared__ long long s_tot;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int wt;
    const int ex = warp_excl_scan(v, lane, wt);
    if (lane == 31) wsum[warp] = wt;
    __syncthreads();
    if (warp == 0) {
        const int x = lane < nw ? wsum[lane] : 0;
        int t;
        const int e = warp_excl_scan(x, lane, t);
        if (lane < nw) wsum[lane] = e;
        if (lane == 0) s_tot = t;
    }
    __syncthreads();
    const long long r = (long long)ex + wsum[warp];
    total = s_tot;
    __syncthreads(); // wsum / s_tot are reused by the next call
    return r;
}

// Exclusive scan over N items, single block.  mode 0: item i = n - depth[i]
// (children of parent i); mode 1: item i = cnt[i].  out[N] = total.
__global__ void __launch_bounds__(kScanThreads) scan_kernel(int mode, const int32_t *depth, int n,
                                                            const int32_t *cnt, const int64_t *N_dev,
                                                            int64_t N_host, int64_t *out)
{
    const int64_t N = N_dev ? *N_dev : N_host;
    long long carry = 0;
    for (int64_t t0 = 0; t0 < N; t0 += blockDim.x) {
        const int64_t i = t0 + threadIdx.x;
        int v = 0;
        if (i < N) v = mode == 0 ? n - depth[i] : cnt[i];
        long long tot;
        const long long ex = block_excl_scan(v, tot);
        if (i < N) out[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) out[N] = carry;
}

// Branching (a7): one warp per parent; children are prefix + j for every
// unscheduled j in ascending order.
__global__ void expand_kernel(const uint16_t *__restrict__ st_pf, const int32_t *__restrict__ st_dp,
                              int64_t first, int64_t B, const int64_t *__restrict__ off,
                              uint16_t *__restrict__ ch_pf, int32_t *__restrict__ ch_dp, int n,
                              int stride)
{
    extern __shared__ uint32_t bm_all[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = (n + 31) >> 5;
    uint32_t *bm = bm_all + wib * nw;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; p < B; p += warps) {
        const uint16_t *row = st_pf + (size_t)(first + p) * stride;
        const int d = st_dp[first + p];
        for (int w = lane; w < nw; w += 32) bm[w] = 0;
        __syncwarp();
        for (int i = lane; i < d; i += 32) atomicOr(&bm[row[i] >> 5], 1u << (row[i] & 31));
        __syncwarp();
        int64_t c = off[p];
        for (int w = 0; w < nw; ++w) {
            uint32_t freeb = ~bm[w];
            if (w == nw - 1 && (n & 31)) freeb &= (1u << (n & 31)) - 1;
            while (freeb) {
                const int j = w * 32 + __ffs(freeb) - 1;
                freeb &= freeb - 1;
                uint16_t *crow = ch_pf + (size_t)c * stride;
                for (int i = lane; i < d; i += 32) crow[i] = row[i];
                if (lane == 0) {
                    crow[d] = (uint16_t)j;
                    ch_dp[c] = d + 1;
                }
                ++c;
            }
        }
        __syncwarp();
    }
}

// Elimination (a6) + leaves (a8): count survivors per block.
__global__ void __launch_bounds__(kPruneThreads)
    prune_kernel(const int32_t *__restrict__ ch_dp, const int32_t *__restrict__ ch_lb,
                 const int64_t *C_dev, int n, const int32_t *inc_dev, unsigned long long *cand,
                 int32_t *bcnt, unsigned long long *stats)
{
    const int64_t C = *C_dev;
    const int inc = *inc_dev;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int survive = 0, pruned = 0, leaf = 0;
    if (i < C) {
        const int d = ch_dp[i], lb = ch_lb[i];
        if (d >= n - 1) { // complete or forced completion: LB is its makespan (R6, P4)
            leaf = 1;
            if (lb < inc) atomicMin(cand, ((unsigned long long)(unsigned)lb << 32) | (unsigned)i);
        } else if (lb < inc) {
            survive = 1;
        } else {
            pruned = 1;
        }
    }
    const int cs = __syncthreads_count(survive);
    const int cp = __syncthreads_count(pruned);
    const int cl = __syncthreads_count(leaf);
    if (threadIdx.x == 0) {
        bcnt[blockIdx.x] = cs;
        if (cp) atomicAdd(&stats[0], (unsigned long long)cp);
        if (cl) atomicAdd(&stats[1], (unsigned long long)cl);
    }
}

// Stream compaction of the survivors onto the stack at `top`, child order.
__global__ void __launch_bounds__(kPruneThreads)
    scatter_kernel(const uint16_t *__restrict__ ch_pf, const int32_t *__restrict__ ch_dp,
                   const int32_t *__restrict__ ch_lb, const int64_t *C_dev, int n, int stride,
                   const int32_t *inc_dev, const int64_t *__restrict__ boff, int64_t top,
                   uint16_t *__restrict__ st_pf, int32_t *__restrict__ st_dp)
{
    __shared__ int64_t s_dst[kPruneThreads];
    __shared__ int64_t s_src[kPruneThreads];
    const int64_t C = *C_dev;
    const int inc = *inc_dev;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int survive = 0, d = 0;
    if (i < C) {
        d = ch_dp[i];
        survive = d < n - 1 && ch_lb[i] < inc;
    }
    long long tot;
    const long long r = block_excl_scan(survive, tot);
    if (survive) {
        s_dst[r] = top + boff[blockIdx.x] + r;
        s_src[r] = i;
        st_dp[top + boff[blockIdx.x] + r] = d;
    }
    __syncthreads();
    // warp-cooperative, coalesced row copies
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    for (int k = wib; k < tot; k += nwb) {
        const uint16_t *src = ch_pf + (size_t)s_src[k] * stride;
        uint16_t *dst = st_pf + (size_t)s_dst[k] * stride;
        const int dd = ch_dp[s_src[k]];
        for (int q = lane; q < dd; q += 32) dst[q] = src[q];
    }
}

// Adopt the best leaf of this iteration (a8) and publish the status.
__global__ void commit_kernel(const uint16_t *__restrict__ ch_pf, const int32_t *__restrict__ ch_dp,
                              int n, int stride, int32_t *inc, unsigned long long *cand,
                              int32_t *perm, long long *packed, int rank, const int64_t *C_dev,
                              const int64_t *T_dev, BBStatus *status)
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
            const uint16_t *row = ch_pf + (size_t)idx * stride;
            const int d = ch_dp[idx];
            for (int w = threadIdx.x; w < (n + 31) / 32; w += blockDim.x) s_bm[w] = 0;
            __syncthreads();
            for (int i = threadIdx.x; i < d; i += blockDim.x) {
                perm[i] = row[i];
                atomicOr(&s_bm[row[i] >> 5], 1u << (row[i] & 31));
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
        status->children = C_dev ? *C_dev : 0;
        status->survivors = T_dev ? *T_dev : 0;
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

void bb_free(BBState *s)
{
    if (!s) return;
    cudaFree(s->st_pf);
    cudaFree(s->st_dp);
    cudaFree(s->ch_pf);
    cudaFree(s->ch_dp);
    cudaFree(s->ch_lb);
    cudaFree(s->off);
    cudaFree(s->boff);
    cudaFree(s->bcnt);
    cudaFree(s->d_inc);
    cudaFree(s->d_cand);
    cudaFree(s->d_packed);
    cudaFree(s->d_scratch);
    cudaFree(s->d_perm);
    cudaFree(s->d_stats);
    cudaFree(s->d_status);
    if (s->h_status) cudaFreeHost(s->h_status);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

int64_t env_i64(const char *name, int64_t dflt)
{
    const char *v = getenv(name);
    return v ? atoll(v) : dflt;
}

// Push nodes given as (depth, prefix) host rows onto the stack top.
int push_host(BBState *s, const std::vector<uint16_t> &pf, const std::vector<int32_t> &dp)
{
    const int64_t k = (int64_t)dp.size();
    if (s->size + k > s->cap) return fsp_fail(FSP_ENOMEM, "B&B stack full");
    cudaError_t e = cudaMemcpyAsync(s->st_pf + (size_t)s->size * s->stride, pf.data(),
                                    sizeof(uint16_t) * pf.size(), cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->st_dp + s->size, dp.data(), sizeof(int32_t) * k,
                            cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B push");
    s->size += k;
    return FSP_OK;
}

// One expand/bound/prune iteration.  Returns FSP_OK (or an error).
int bb_iterate(BBState *s)
{
    const fsp_instance *inst = s->inst;
    const int n = s->n, stride = s->stride;
    cudaStream_t st = s->stream;
    const int64_t open = s->size - s->base;
    if (open <= 0) return FSP_OK;
    // selection: the top B nodes (deepest-first batch), sized from the last
    // iteration's children per parent so the child pool fills the GPU; the
    // exact child count is checked after the scan and B halved if it overflows
    const double kpp = std::max(1.0, std::min((double)n, s->kids_per_parent));
    int64_t B = std::min<int64_t>(open, std::max<int64_t>(1, (int64_t)(s->ccap / kpp)));
    // beam width of the depth-first batches: B parents per level with ~n/2
    // children each over n levels must fit the stack (B * n^2/2 <= cap)
    B = std::min<int64_t>(B, std::max<int64_t>(1, s->cap / std::max<int64_t>(1, (int64_t)n * n / 2)));
    // keep n*n slots of headroom: from any state a depth-first descent (B = 1)
    // needs at most n children per level for n levels, so the search never
    // dead-ends on memory
    const int64_t usable = s->cap - (int64_t)n * n;
    int64_t first = 0;
    for (;;) {
        first = s->size - B;
        scan_kernel<<<1, kScanThreads, 0, st>>>(0, s->st_dp + first, n, nullptr, nullptr, B, s->off);
        cudaError_t e = cudaMemcpyAsync(&s->h_status->children, s->off + B, 8,
                                        cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B scan");
        const long long C = s->h_status->children;
        // the children must fit the child buffer, and (all surviving) the stack
        const int64_t room = std::max<int64_t>(0, std::min<int64_t>(s->ccap, usable - first));
        if (C <= room) break;
        if (B == 1) {
            if (first + C > s->cap || C > s->ccap) return fsp_fail(FSP_ENOMEM, "B&B stack full");
            break;
        }
        B = std::max<int64_t>(1, std::min<int64_t>(B / 2, (int64_t)((double)B * room / (double)C * 0.9)));
    }
    s->size = first;
    const int64_t maxC = s->h_status->children;

    const int ewarps = 8;
    const int eblocks = (int)std::min<int64_t>((B + ewarps - 1) / ewarps, 148 * 16);
    expand_kernel<<<eblocks, ewarps * 32, ewarps * ((n + 31) / 32) * 4, st>>>(
        s->st_pf, s->st_dp, first, B, s->off, s->ch_pf, s->ch_dp, n, stride);
    const int64_t *C_dev = s->off + B;
    int rc = fsp_launch_lb_dev(inst, s->ch_pf, stride, s->ch_dp, maxC, C_dev, s->ch_lb, st);
    if (rc != FSP_OK) return rc;
    const int nblk = (int)((maxC + kPruneThreads - 1) / kPruneThreads);
    prune_kernel<<<nblk, kPruneThreads, 0, st>>>(s->ch_dp, s->ch_lb, C_dev, n, s->d_inc, s->d_cand,
                                                  s->bcnt, s->d_stats);
    scan_kernel<<<1, kScanThreads, 0, st>>>(1, nullptr, n, s->bcnt, nullptr, nblk, s->boff);
    scatter_kernel<<<nblk, kPruneThreads, 0, st>>>(s->ch_pf, s->ch_dp, s->ch_lb, C_dev, n, stride,
                                                    s->d_inc, s->boff, first, s->st_pf, s->st_dp);
    commit_kernel<<<1, 256, 0, st>>>(s->ch_pf, s->ch_dp, n, stride, s->d_inc, s->d_cand, s->d_perm,
                                     s->d_packed, s->rank, C_dev, s->boff + nblk, s->d_status);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->h_status, s->d_status, sizeof(BBStatus), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B iteration");
    s->size = first + s->h_status->survivors;
    s->stats.bounded += s->h_status->children;
    s->stats.branched += B;
    s->stats.iterations += 1;
    if (s->h_status->improved) {
        s->have = 1;
        s->perm_ms = s->h_status->incumbent;
    }
    if (B > 0 && s->h_status->children > 0)
        s->kids_per_parent = (double)s->h_status->children / (double)B;
    return FSP_OK;
}

int bb_create(const fsp_instance *inst, int32_t initial_ub, int32_t rank, int32_t world,
              void *stream, BBState **out)
{
    if (!inst || !out || world < 1 || rank < 0 || rank >= world || initial_ub < 0)
        return fsp_fail(FSP_EINVAL, "bad B&B arguments");
    BBState *s = new (std::nothrow) BBState();
    if (!s) return fsp_fail(FSP_ENOMEM, "host allocation");
    s->inst = inst;
    s->rank = rank;
    s->world = world;
    s->n = inst->n;
    s->stride = (inst->n + 7) & ~7;
    s->initial_inc = initial_ub == INT32_MAX ? INT32_MAX : initial_ub + 1; // R9
    cudaError_t e = cudaSuccess;
    if (stream) {
        s->stream = static_cast<cudaStream_t>(stream);
    } else {
        e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        s->own_stream = true;
    }
    const int n = s->n;
    const size_t rec = (size_t)s->stride * 2 + 4;
    size_t freeb = 0, totalb = 0;
    if (e == cudaSuccess) e = cudaMemGetInfo(&freeb, &totalb);
    // child buffer: enough children to fill the GPU several times over
    s->ccap = env_i64("FSP_BB_CHILDREN", std::max<int64_t>(1 << 22, (int64_t)n * 4));
    s->kids_per_parent = n;
    // the stack may take most of the free HBM (180 GB per B200): its size bounds
    // the beam width of the depth-first batches (see bb_iterate)
    const double frac = getenv("FSP_BB_MEM_FRAC") ? atof(getenv("FSP_BB_MEM_FRAC")) : 0.6;
    int64_t cap = (int64_t)((double)freeb * frac / rec);
    cap = env_i64("FSP_BB_STACK", std::min<int64_t>(cap, (int64_t)1 << 31));
    s->cap = std::max<int64_t>(cap, (int64_t)n * n * 4);
    const int64_t maxB = s->ccap; // parents per iteration never exceed the children
    const int64_t nblk = (s->ccap + kPruneThreads - 1) / kPruneThreads + 1;
    auto alloc = [&](void **p, size_t bytes) {
        if (e == cudaSuccess) e = cudaMalloc(p, bytes);
    };
    alloc((void **)&s->st_pf, (size_t)s->cap * s->stride * 2);
    alloc((void **)&s->st_dp, (size_t)s->cap * 4);
    alloc((void **)&s->ch_pf, (size_t)s->ccap * s->stride * 2);
    alloc((void **)&s->ch_dp, (size_t)s->ccap * 4);
    alloc((void **)&s->ch_lb, (size_t)s->ccap * 4);
    alloc((void **)&s->off, (size_t)(maxB + 1) * 8);
    alloc((void **)&s->boff, (size_t)(nblk + 1) * 8);
    alloc((void **)&s->bcnt, (size_t)nblk * 4);
    alloc((void **)&s->d_inc, 4);
    alloc((void **)&s->d_cand, 8);
    alloc((void **)&s->d_packed, 8);
    alloc((void **)&s->d_scratch, 8);
    alloc((void **)&s->d_perm, (size_t)n * 4);
    alloc((void **)&s->d_stats, 16);
    alloc((void **)&s->d_status, sizeof(BBStatus));
    if (e == cudaSuccess) e = cudaMallocHost((void **)&s->h_status, sizeof(BBStatus));
    if (e == cudaSuccess) e = cudaMemcpy(s->d_inc, &s->initial_inc, 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(s->d_cand, 0xff, 8);
    if (e == cudaSuccess) e = cudaMemset(s->d_stats, 0, 16);
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
    if (world == 1) {
        pf.assign(s->stride, 0xffff);
        dp.push_back(0);
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
    unsigned long long h[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(h, s->d_stats, 16, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B stats");
    s->stats.pruned = (int64_t)h[0];
    s->stats.leaves = (int64_t)h[1];
    return FSP_OK;
}

int result(BBState *s, int32_t *makespan_out, int32_t *perm_out)
{
    int32_t inc = 0;
    cudaError_t e = cudaMemcpyAsync(&inc, s->d_inc, 4, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess && perm_out && s->have)
        e = cudaMemcpyAsync(perm_out, s->d_perm, sizeof(int32_t) * s->n, cudaMemcpyDeviceToHost,
                            s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "B&B result");
    (void)inc;
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

extern "C" int fsp_bb_init(const fsp_instance *inst, int32_t initial_ub, int32_t rank,
                           int32_t world, void **state)
{
    if (!state) return fsp_fail(FSP_EINVAL, "null state");
    BBState *s = nullptr;
    int rc = bb_create(inst, initial_ub, rank, world, nullptr, &s);
    *state = s;
    return rc;
}

extern "C" int fsp_bb_step(void *state, int32_t iters, void *)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || iters < 0) return fsp_fail(FSP_EINVAL, "bad B&B state");
    for (int i = 0; i < iters && s->size > s->base; ++i) {
        int rc = bb_iterate(s);
        if (rc != FSP_OK) return rc;
    }
    return read_stats(s);
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
    return s ? (int64_t)s->stride * 2 + 4 : 0;
}

// Donor side: the shallowest open nodes (bottom of the stack, largest
// subtrees) go out as [k][stride] u16 prefixes followed by [k] int32 depths.
extern "C" int fsp_bb_export(void *state, int64_t max_nodes, void *d_buf, int64_t *n_out)
{
    BBState *s = static_cast<BBState *>(state);
    if (!s || !n_out || max_nodes < 0 || (max_nodes > 0 && !d_buf))
        return fsp_fail(FSP_EINVAL, "bad export arguments");
    const int64_t k = std::min(max_nodes, s->size - s->base);
    *n_out = k;
    if (k == 0) return FSP_OK;
    uint8_t *b = static_cast<uint8_t *>(d_buf);
    cudaError_t e = cudaMemcpyAsync(b, s->st_pf + (size_t)s->base * s->stride,
                                    (size_t)k * s->stride * 2, cudaMemcpyDeviceToDevice, s->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(b + (size_t)k * s->stride * 2, s->st_dp + s->base, (size_t)k * 4,
                            cudaMemcpyDeviceToDevice, s->stream);
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
    // compact the deque first if the bottom has drifted
    if (s->base > 0) {
        const int64_t open = s->size - s->base;
        cudaError_t e = cudaSuccess;
        if (open > 0) {
            // move in chunks that never overlap destructively (dst < src)
            for (int64_t q = 0; q < open && e == cudaSuccess; q += s->base) {
                const int64_t c = std::min(s->base, open - q);
                e = cudaMemcpyAsync(s->st_pf + (size_t)q * s->stride,
                                    s->st_pf + (size_t)(s->base + q) * s->stride,
                                    (size_t)c * s->stride * 2, cudaMemcpyDeviceToDevice, s->stream);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(s->st_dp + q, s->st_dp + s->base + q, (size_t)c * 4,
                                        cudaMemcpyDeviceToDevice, s->stream);
            }
        }
        if (e != cudaSuccess) return fsp_cuda_fail(e, "import compaction");
        s->size = open;
        s->base = 0;
    }
    if (s->size + k > s->cap) return fsp_fail(FSP_ENOMEM, "B&B stack full");
    const uint8_t *b = static_cast<const uint8_t *>(d_buf);
    cudaError_t e = cudaMemcpyAsync(s->st_pf + (size_t)s->size * s->stride, b,
                                    (size_t)k * s->stride * 2, cudaMemcpyDeviceToDevice, s->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(s->st_dp + s->size, b + (size_t)k * s->stride * 2, (size_t)k * 4,
                            cudaMemcpyDeviceToDevice, s->stream);
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
