// wpn.cu — the north_star's work mapping, measured against the product kernel
// ("A/B: warp per sub-problem"): one warp per sub-problem, lanes
// over machine couples, heads/tails/loads by lanes over jobs with warp
// reductions.  Same bound as lb_kernel.cu (Fig. 3, readings R1-R6),
// int32 arithmetic, selected with FSP_LB_MAPPING=warp at instance load
// (fsp_launch_lb routes the dense pools here; B&B pools are unaffected).
//
// Per CTA iteration a batch of WPN_WARPS x WPN_NPW nodes:
//   A. per node (its warp): the prefix staged in shared memory, the
//      unscheduled flags (one byte per job), the completion times C_k by a
//      systolic pass (lane k = machine k, job i at step i + k, C_k-1 from lane
//      k-1 by shfl.up), then the heads r_jk (R3), tails q_jl (R4) and loads
//      L_k with lane = job, reduced over the warp (REDUX min / add);
//   B. per group of 32 couples (records [position][32 couples] staged by the
//      whole CTA): lane = couple, the walk e <- max(e + x_j, y_j) over the
//      couple's Johnson order for every node of the warp (the flag byte of
//      job j gates the update), then a warp max.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <numeric>
#include <vector>

#include "fsp_internal.h"

namespace {

constexpr int WPN_WARPS = 8;  // warps per CTA
constexpr int WPN_NPW = 4;    // nodes per warp per batch
constexpr int WPN_NB = WPN_WARPS * WPN_NPW;

struct WpnArgs {
    const int32_t *ptm;       // [n][m] int32 (global; staged)
    const int2 *recs;         // [groups][nrec][32] {y, (x << 16) | j}
    const uint16_t *prefix;
    const int32_t *depth;
    int32_t *lb_out;
    int *err;
    long long pool;
    int n, m, P, groups, nrec, stride, flag_bytes;
};

// shared memory: ptm [n][m] int32 | records of one group [nrec][32] int2 |
// per node of the batch: flags [flag_bytes] u8, R/A/Q [3][32] int32 | per warp:
// the node's prefix [n] u16
template <int MAXM>
__global__ void __launch_bounds__(WPN_WARPS * 32) lb_wpn_kernel(const WpnArgs a)
{
    extern __shared__ __align__(16) uint8_t smem[];
    const int n = a.n, m = a.m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t *s_ptm = reinterpret_cast<int32_t *>(smem);
    int2 *s_rec = reinterpret_cast<int2 *>(smem + (((size_t)n * m * 4 + 15) & ~size_t(15)));
    uint8_t *s_node = reinterpret_cast<uint8_t *>(s_rec + (size_t)a.nrec * 32);
    const size_t node_bytes = (size_t)a.flag_bytes + 3 * 32 * 4;
    uint16_t *s_pf = reinterpret_cast<uint16_t *>(s_node + WPN_NB * node_bytes) + (size_t)warp * ((n + 7) & ~7);

    for (int i = threadIdx.x; i < n * m; i += blockDim.x) s_ptm[i] = a.ptm[i];
    __syncthreads();

    const long long nbatch = (a.pool + WPN_NB - 1) / WPN_NB;
    for (long long b = blockIdx.x; b < nbatch; b += gridDim.x) {
        int lbv[WPN_NPW];
        bool bad = false;
        // ---------------- A: per node of this warp ----------------
        for (int t = 0; t < WPN_NPW; ++t) {
            lbv[t] = 0; // R1: the max over couples starts at 0
            const long long node = b * WPN_NB + warp * WPN_NPW + t;
            uint8_t *fl = s_node + (size_t)(warp * WPN_NPW + t) * node_bytes;
            int32_t *st = reinterpret_cast<int32_t *>(fl + a.flag_bytes); // R[32] A[32] Q[32]
            const bool has = node < a.pool;
            int d = has ? a.depth[node] : n; // absent nodes: complete (all flags 0)
            if (d < 0 || d > n || d > a.stride) {
                bad = true;
                d = 0;
            }
            for (int j = lane; j < a.flag_bytes; j += 32) fl[j] = j < n && has ? 1 : 0;
            __syncwarp();
            const uint16_t *row = a.prefix + (size_t)(has ? node : 0) * a.stride;
            for (int i = lane; i < d; i += 32) {
                uint32_t j = has ? row[i] : 0u;
                if (j >= (uint32_t)n) {
                    bad = true;
                    j = 0;
                }
                s_pf[i] = (uint16_t)j;
                fl[j] = 0;
            }
            __syncwarp();
            // C_k systolic: lane k holds C_k; at step s it takes job
            // i = s - k with C_k-1 of the same job from lane k-1 (its step s-1)
            int C = 0, out = 0;
            if (has) {
                for (int s = 0; s < d + m - 1; ++s) {
                    const int up = __shfl_up_sync(0xffffffffu, out, 1);
                    const int i = s - lane;
                    if (lane < m && i >= 0 && i < d) {
                        C = max(C, lane ? up : 0) + s_ptm[s_pf[i] * m + lane];
                        out = C;
                    }
                }
            }
            // heads / tails / loads, lane = job (R3, R4, R5), then reductions
            int Rm[MAXM], Qm[MAXM], Lk[MAXM], Cb[MAXM];
#pragma unroll
            for (int k = 0; k < MAXM; ++k) {
                Cb[k] = __shfl_sync(0xffffffffu, C, k);
                Rm[k] = Qm[k] = INT_MAX;
                Lk[k] = 0;
            }
            int cnt = 0;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const int j = j0 + lane;
                if (j < n && fl[j]) {
                    ++cnt;
                    const int32_t *p = s_ptm + (size_t)j * m;
                    int r = Cb[0];
#pragma unroll
                    for (int k = 0; k < MAXM; ++k) {
                        if (k < m) {
                            if (k) r = max(Cb[k], r + p[k - 1]);
                            Rm[k] = min(Rm[k], r);
                            Lk[k] += p[k];
                        }
                    }
                    int q = 0;
#pragma unroll
                    for (int l = MAXM - 1; l >= 0; --l) {
                        if (l < m) {
                            Qm[l] = min(Qm[l], q);
                            q += p[l];
                        }
                    }
                }
            }
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (has && cnt != n - d) bad = true; // repeated job
#pragma unroll
            for (int k = 0; k < MAXM; ++k) {
                if (k < m) {
                    const int R = (int)__reduce_min_sync(0xffffffffu, (unsigned)Rm[k]);
                    const int Q = (int)__reduce_min_sync(0xffffffffu, (unsigned)Qm[k]);
                    const int L = (int)__reduce_add_sync(0xffffffffu, (unsigned)Lk[k]);
                    if (lane == k) {
                        if (cnt == 0) { // R6: complete schedule
                            st[k] = st[32 + k] = Cb[k];
                            st[64 + k] = 0;
                        } else {
                            st[k] = R;
                            st[32 + k] = R + L;
                            st[64 + k] = Q;
                        }
                    }
                }
            }
        }
        if (bad) atomicOr(a.err, 1);
        // ---------------- B: couple groups, lane = couple ----------------
        for (int g = 0; g < a.groups; ++g) {
            __syncthreads(); // every warp is done with the previous group
            {
                const int4 *src = reinterpret_cast<const int4 *>(a.recs + (size_t)g * a.nrec * 32);
                int4 *dst = reinterpret_cast<int4 *>(s_rec);
                for (int i = threadIdx.x; i < a.nrec * 16; i += blockDim.x) dst[i] = src[i];
            }
            __syncthreads();
            const int c = g * 32 + lane; // this lane's couple (k, l), k < l
            int k = 0, l = 1;
            if (c < a.P) {
                int rem = c;
                while (rem >= m - 1 - k) {
                    rem -= m - 1 - k;
                    ++k;
                }
                l = k + 1 + rem;
            }
            for (int t = 0; t < WPN_NPW; ++t) {
                const uint8_t *fl = s_node + (size_t)(warp * WPN_NPW + t) * node_bytes;
                const int32_t *st = reinterpret_cast<const int32_t *>(fl + a.flag_bytes);
                int e = st[l] - st[k]; // lines 06-07: t2 - t1 at R_l - R_k
                const int2 *r = s_rec + lane;
#pragma unroll 4
                for (int i = 0; i < a.nrec; ++i) {
                    const int2 v = r[(size_t)i * 32];
                    if (fl[v.y & 0xffff]) e = max(e + (v.y >> 16), v.x); // lines 10-15
                }
                const int val = c < a.P ? e + st[32 + k] + st[64 + l] : 0; // lines 18-19
                lbv[t] = max(lbv[t], (int)__reduce_max_sync(0xffffffffu, (unsigned)val));
            }
        }
        for (int t = 0; t < WPN_NPW; ++t) {
            const long long node = b * WPN_NB + warp * WPN_NPW + t;
            if (lane == 0 && node < a.pool) a.lb_out[node] = lbv[t];
        }
    }
}

size_t wpn_smem(int n, int m, int nrec)
{
    const size_t flag_bytes = ((size_t)n + 1 + 15) & ~size_t(15);
    return (((size_t)n * m * 4 + 15) & ~size_t(15)) + (size_t)nrec * 32 * 8 +
           WPN_NB * (flag_bytes + 3 * 32 * 4) + (size_t)WPN_WARPS * ((n + 7) & ~7) * 2;
}

} // namespace

// Records [group][position][32 couples] {y, (x << 16) | j} in each couple's
// Johnson-with-lags order (instance.cu's rule, rebuilt here: this file stands
// alone); couples past P and positions past n point at job n (flag 0).
int fsp_wpn_build(fsp_instance *inst)
{
    const int n = inst->n, m = inst->m, P = inst->P;
    if (m > 32) return fsp_fail(FSP_ERANGE, "warp-per-node mapping: m > 32");
    const int groups = (P + 31) / 32, nrec = n;
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, inst->device);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "device attribute");
    if (wpn_smem(n, m, nrec) > (size_t)optin) return fsp_fail(FSP_ERANGE, "warp-per-node mapping: smem");
    std::vector<int2> recs((size_t)groups * nrec * 32, make_int2(0, n));
    const int32_t *ptm = inst->h_ptm;
    std::vector<int> order(n), A(n), B(n);
    int c = 0;
    for (int k = 0; k < m; ++k) {
        for (int l = k + 1; l < m; ++l, ++c) {
            for (int j = 0; j < n; ++j) {
                int a = 0, b = 0;
                for (int i = k; i < l; ++i) a += ptm[(size_t)j * m + i];     // p_jk + lag
                for (int i = k + 1; i <= l; ++i) b += ptm[(size_t)j * m + i]; // lag + p_jl
                A[j] = a;
                B[j] = b;
            }
            std::iota(order.begin(), order.end(), 0);
            std::sort(order.begin(), order.end(), [&](int x, int y) {
                const bool fx = A[x] <= B[x], fy = A[y] <= B[y];
                if (fx != fy) return fx;
                if (fx ? A[x] != A[y] : B[x] != B[y]) return fx ? A[x] < A[y] : B[x] > B[y];
                return x < y;
            });
            for (int i = 0; i < n; ++i) {
                const int j = order[i];
                const int x = ptm[(size_t)j * m + l] - ptm[(size_t)j * m + k];
                recs[((size_t)(c / 32) * nrec + i) * 32 + c % 32] =
                    make_int2(B[j], (int)(((uint32_t)x << 16) | (uint32_t)j));
            }
        }
    }
    e = cudaMalloc(&inst->d_wpn, recs.size() * sizeof(int2));
    if (e == cudaSuccess) e = cudaMemcpy(inst->d_wpn, recs.data(), recs.size() * sizeof(int2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "warp-per-node tables");
    e = cudaFuncSetAttribute(lb_wpn_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(lb_wpn_kernel<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(lb_wpn_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "cudaFuncSetAttribute");
    inst->wpn = true;
    return FSP_OK;
}

int fsp_launch_lb_wpn(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                      const int32_t *depth, int64_t pool, int32_t *lb_out, cudaStream_t s)
{
    WpnArgs a;
    a.ptm = inst->d_ptm32;
    a.recs = reinterpret_cast<const int2 *>(inst->d_wpn);
    a.prefix = prefix;
    a.depth = depth;
    a.lb_out = lb_out;
    a.err = inst->d_err;
    a.pool = pool;
    a.n = inst->n;
    a.m = inst->m;
    a.P = inst->P;
    a.groups = (inst->P + 31) / 32;
    a.nrec = inst->n;
    a.stride = stride;
    a.flag_bytes = (int)(((size_t)inst->n + 1 + 15) & ~size_t(15));
    const size_t sm = wpn_smem(a.n, a.m, a.nrec);
    auto kern = a.m <= 8 ? lb_wpn_kernel<8> : a.m <= 20 ? lb_wpn_kernel<20> : lb_wpn_kernel<32>;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPN_WARPS * 32, sm);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "occupancy");
    const long long nbatch = (pool + WPN_NB - 1) / WPN_NB;
    const int grid = (int)std::min<long long>(nbatch, (long long)std::max(1, per_sm) * inst->plan.num_sms);
    kern<<<grid, WPN_WARPS * 32, sm, s>>>(a);
    e = cudaGetLastError();
    return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "lb_wpn_kernel launch");
}
