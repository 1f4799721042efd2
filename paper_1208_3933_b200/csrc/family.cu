// family.cu — sibling-incremental bounding: the LBs of
// a parent's children from ONE pass over the parent's unscheduled set per
// couple, instead of one couple walk per child.
//
// Fig. 3 lines 08-17 walk the unscheduled jobs of a node in the
// couple's Johnson-with-lags order; in the difference form
// every job j is the map f_j(e) = max(e + x_j, y_j), x_j = p_jl - p_jk,
// y_j = lag_j + p_jl.  Maps of this form compose in closed form:
//     (A2, B2) o (A1, B1) : e -> max(e + A1 + A2, max(B1 + A2, B2)),
// the identity being (0, -inf).  A child x of a parent with unscheduled set S
// walks S \ {x}; its map is Suf(x) o Pre(x), the compositions of the jobs of S
// after and before x in the couple's order.  One forward pass (prefixes) and
// one backward pass (suffixes) over S give every child's couple value in O(1):
//     A = A_pre + A_suf,  B = max(B_pre + A_suf, B_suf),
//     value = max(R'_l - R'_k + A, B) + (R'_k + L'_k) + Q'_l
// with the child's own heads R', loads L' and tails Q' (Fig. 3 lines 06-07,
// 18-19).  Only integer additions are regrouped: bit-identical to Fig. 3.
//
// Mapping: one warp per parent (|S| = n - d <= 32, n <= 256).  Heads: lane t
// = child t (loop over S).  Couples: lane c = couple c (rounds of 32); each
// lane sorts S into its couple's order through the inverse position table
// (positions set in a per-lane bitmask, read back in order), then runs the
// two passes; per-(child, lane) partial maxima are reduced at the end.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "fsp_internal.h"

namespace {

constexpr int kNeg = INT_MIN / 4; // -inf of the compositions (no overflow)
constexpr int kFamWarps = 8;      // most warps per CTA (shared memory permitting)

struct FamArgs {
    const uint8_t *blob; // fam_blob layout (fsp_fam_layout)
    fsp_fam_layout L;
    int n, m, P;
    // parents
    const uint16_t *ppf;  // parent prefixes [B][stride]
    int stride;
    const int32_t *pdp;   // parent depths [B]
    const int32_t *pC;    // parent completion times [B][m] (nullable: from the prefix)
    int64_t B;
    // children: B&B mode (off != nullptr): parent p's children are
    // [off[p], off[p+1]) (low 32 bits), child c's job in ckey[c] & 0xfff and
    // its LB goes to out[c]; ABI mode: all unscheduled jobs of the parent in
    // ascending order, LB of the t-th to out[p * 32 + t]
    const int64_t *off;
    const unsigned long long *ckey;
    int32_t *out;
    const int *flag; // B&B: the batch takes this kernel (else exit)
};

template <int MAXM>
__global__ void __launch_bounds__(kFamWarps * 32) family_kernel(const FamArgs a)
{
    if (a.flag && *a.flag == 0) return;
    extern __shared__ __align__(16) uint8_t fsm[];
    const int n = a.n, m = a.m, P = a.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    // tables, staged once per CTA: couples (k | l << 16), inverse positions
    // pos[c][j], Johnson orders jm[c][pos], (p_jk, sum_{i<=k} p_ji) per job,
    // tails q_jk = sum_{i>k} p_ji
    for (size_t i = threadIdx.x * 16; i < a.L.table_bytes; i += blockDim.x * 16)
        *reinterpret_cast<uint4 *>(fsm + i) = *reinterpret_cast<const uint4 *>(a.blob + i);
    __syncthreads();
    const uint32_t *kl = reinterpret_cast<const uint32_t *>(fsm + a.L.off_kl);
    const uint8_t *ipos = fsm + a.L.off_pos;
    const uint8_t *jm = fsm + a.L.off_jm;
    const int2 *pc = reinterpret_cast<const int2 *>(fsm + a.L.off_pc);
    const int *qt = reinterpret_cast<const int *>(fsm + a.L.off_q);
    // per-warp scratch
    uint8_t *ws = fsm + a.L.table_bytes + (size_t)warp * a.L.warp_bytes;
    int *preA = reinterpret_cast<int *>(ws);          // [32 children][32 lanes]
    int *preB = preA + 32 * 32;
    int *part = preB + 32 * 32;                       // partial maxima [32][32]
    uint32_t *bm = reinterpret_cast<uint32_t *>(part + 32 * 32); // [8 words][32 lanes]
    int *Rp = reinterpret_cast<int *>(bm + 8 * 32);  // [32][m]: R'_k
    int *Ap = Rp + 32 * m;                            // [32][m]: R'_k + L'_k
    int *Qp = Ap + 32 * m;                            // [32][m]: Q'_l
    uint32_t *sched = reinterpret_cast<uint32_t *>(Qp + 32 * m); // [8]
    uint8_t *slot = reinterpret_cast<uint8_t *>(sched + 8);      // [n]: child slot of job j

    const int64_t warps = (int64_t)gridDim.x * W;
    for (int64_t p = (int64_t)blockIdx.x * W + warp; p < a.B; p += warps) {
        const int d = a.pdp[p];
        const int np = n - d; // |S| <= 32 (checked by the caller)
        int64_t c0 = (int64_t)p * 32;
        int g = np;
        if (a.off) {
            c0 = a.off[p] & 0xffffffffll;
            g = (int)((a.off[p + 1] & 0xffffffffll) - c0);
        }
        if (g <= 0 || np <= 0 || np > 32) continue; // (np: R6 leaves are bounded as children)
        // ---- S: the parent's unscheduled jobs, lane t < np holds the t-th
        const uint16_t *row = a.ppf + (size_t)p * a.stride;
        if (lane < 8) sched[lane] = 0;
        __syncwarp();
        for (int i = lane; i < d; i += 32) {
            const uint32_t j = row[i];
            atomicOr(&sched[j >> 5], 1u << (j & 31));
        }
        __syncwarp();
        int sj = -1;
        {
            int base = 0;
            for (int w = 0; w * 32 < n; ++w) {
                uint32_t fr = ~sched[w];
                if (w * 32 + 32 > n) fr &= (1u << (n - w * 32)) - 1u;
                const int c = __popc(fr);
                if (lane >= base && lane < base + c) sj = w * 32 + (int)__fns(fr, 0, lane - base + 1);
                base += c;
            }
        }
        // ---- parent completion times: given, or from the prefix
        int Cp[MAXM];
#pragma unroll
        for (int k = 0; k < MAXM; ++k) Cp[k] = 0;
        if (a.pC) {
#pragma unroll
            for (int k = 0; k < MAXM; ++k)
                if (k < m) Cp[k] = a.pC[(size_t)p * m + k];
        } else {
            for (int i = 0; i < d; ++i) {
                const int j = row[i];
                int prev = 0;
#pragma unroll
                for (int k = 0; k < MAXM; ++k)
                    if (k < m) {
                        Cp[k] = max(Cp[k], prev) + pc[j * m + k].x;
                        prev = Cp[k];
                    }
            }
        }
        // ---- children: lane t < g owns child t (job xt), slot map job -> t
        int xt = -1;
        if (lane < g) xt = a.off ? (int)(a.ckey[c0 + lane] & 0xfffu) : sj;
        if (lane < np) slot[sj] = 0xff;
        __syncwarp();
        if (lane < g) slot[xt] = (uint8_t)lane;
        for (int i = lane; i < 32 * 32; i += 32) part[i] = 0; // R1: the max starts at 0
        __syncwarp();
        // ---- a1-a3 per child: C' = C + x (one step), heads R', loads L', tails Q'
        {
            const bool own = lane < g;
            int Cc[MAXM], R[MAXM], Lc[MAXM], Q[MAXM];
            int prev = 0;
#pragma unroll
            for (int k = 0; k < MAXM; ++k) {
                if (k < m) {
                    Cc[k] = max(Cp[k], prev) + (own ? pc[xt * m + k].x : 0);
                    prev = Cc[k];
                }
                R[k] = INT_MAX;
                Q[k] = INT_MAX;
                Lc[k] = 0;
            }
            for (int i = 0; i < np; ++i) {
                const int j = __shfl_sync(0xffffffffu, sj, i);
                if (!own || j == xt) continue;
                // r_j0 = C'_0, r_jk = max(C'_k, r_j,k-1 + p_j,k-1) (R3); R_k = min
                int r = Cc[0];
#pragma unroll
                for (int k = 0; k < MAXM; ++k) {
                    if (k < m) {
                        const int pk = pc[j * m + k].x;
                        if (k > 0) r = max(Cc[k], r);
                        R[k] = min(R[k], r);
                        r += pk;
                        Lc[k] += pk;
                        Q[k] = min(Q[k], qt[j * m + k]);
                    }
                }
            }
            if (np == 1) { // R6: the child is a complete schedule
#pragma unroll
                for (int k = 0; k < MAXM; ++k) {
                    R[k] = Cc[k];
                    Q[k] = 0;
                    Lc[k] = 0;
                }
            }
            if (own) {
#pragma unroll
                for (int k = 0; k < MAXM; ++k) {
                    if (k < m) {
                        Rp[lane * m + k] = R[k];
                        Ap[lane * m + k] = R[k] + Lc[k];
                        Qp[lane * m + k] = Q[k];
                    }
                }
            }
        }
        __syncwarp();
        // ---- a4-a5: couples, lane c = couple c
        for (int cr = 0; cr < P; cr += 32) {
            const int c = cr + lane;
            const bool act = c < P;
            const uint32_t kv = act ? kl[c] : 0u;
            const int k = kv & 0xffff, l = kv >> 16;
#pragma unroll
            for (int w = 0; w < 8; ++w) bm[w * 32 + lane] = 0;
            // S in this couple's order: set each job's position
            for (int i = 0; i < np; ++i) {
                const int j = __shfl_sync(0xffffffffu, sj, i);
                if (act) {
                    const int pos = ipos[(size_t)c * n + j];
                    bm[(pos >> 5) * 32 + lane] |= 1u << (pos & 31);
                }
            }
            if (act) {
                // forward: compositions of the jobs before each child
                int A = 0, B = kNeg, w = 0;
                uint32_t bits = bm[lane];
                for (int i = 0; i < np; ++i) {
                    while (!bits) bits = bm[(++w) * 32 + lane];
                    const int pos = w * 32 + __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int j = jm[(size_t)c * n + pos];
                    const int t = slot[j];
                    const int2 vk = pc[j * m + k], vl = pc[j * m + l];
                    const int x = vl.x - vk.x, y = vl.y - vk.y;
                    if (t != 0xff) {
                        preA[t * 32 + lane] = A;
                        preB[t * 32 + lane] = B;
                    }
                    A += x;
                    B = max(B + x, y);
                }
                // backward: compositions of the jobs after each child, combined
                A = 0;
                B = kNeg;
                w = 7;
                bits = bm[7 * 32 + lane];
                for (int i = 0; i < np; ++i) {
                    while (!bits) bits = bm[(--w) * 32 + lane];
                    const int hb = 31 - __clz(bits);
                    const int pos = w * 32 + hb;
                    bits &= ~(1u << hb);
                    const int j = jm[(size_t)c * n + pos];
                    const int t = slot[j];
                    const int2 vk = pc[j * m + k], vl = pc[j * m + l];
                    const int x = vl.x - vk.x, y = vl.y - vk.y;
                    if (t != 0xff) {
                        const int Ac = preA[t * 32 + lane] + A;
                        const int Bc = max(preB[t * 32 + lane] + A, B);
                        const int e0 = Rp[t * m + l] - Rp[t * m + k];
                        const int v = max(e0 + Ac, Bc) + Ap[t * m + k] + Qp[t * m + l];
                        part[t * 32 + lane] = max(part[t * 32 + lane], v);
                    }
                    B = max(y + A, B);
                    A += x;
                }
            }
            __syncwarp();
        }
        // ---- LB of child t = max over couples (lanes)
        if (lane < g) {
            int lb = 0;
            for (int u = 0; u < 32; ++u) lb = max(lb, part[lane * 32 + ((u + lane) & 31)]);
            if (np == 1) lb = Rp[lane * m + (m - 1)]; // R6: the makespan
            a.out[c0 + lane] = lb;
        }
        __syncwarp();
    }
}

template <int MAXM>
int launch_family(const fsp_instance *inst, const FamArgs &a, cudaStream_t s)
{
    const fsp_fam_layout &L = inst->fam;
    const size_t smem = L.table_bytes + (size_t)L.warps * L.warp_bytes;
    static bool attr_set = false;
    if (!attr_set) {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, inst->device);
        cudaError_t e = cudaFuncSetAttribute(family_kernel<MAXM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             optin);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "family attribute");
        attr_set = true;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, inst->device);
    family_kernel<MAXM><<<sms, L.warps * 32, smem, s>>>(a);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "family_kernel launch");
}

} // namespace

// Host-side tables (once per instance; independent of the lb kernel's):
// [kl u32 x P][pos u8 x P x n][jm u8 x P x n][(p, cum) int2 x n x m][q int32 x n x m]
int fsp_fam_build(fsp_instance *inst)
{
    const int n = inst->n, m = inst->m, P = inst->P;
    inst->fam = fsp_fam_layout{};
    if (n > 256 || getenv("FSP_NO_FAMILY")) return FSP_OK; // u8 positions and jobs
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    fsp_fam_layout L{};
    L.off_kl = 0;
    L.off_pos = al((size_t)P * 4);
    L.off_jm = al(L.off_pos + (size_t)P * n);
    L.off_pc = al(L.off_jm + (size_t)P * n);
    L.off_q = al(L.off_pc + (size_t)n * m * 8);
    L.table_bytes = al(L.off_q + (size_t)n * m * 4);
    L.warp_bytes = al((size_t)3 * 32 * 32 * 4 + 8 * 32 * 4 + (size_t)3 * 32 * m * 4 + 8 * 4 + (size_t)n);
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, inst->device);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "device attribute");
    L.warps = 0;
    for (int w = kFamWarps; w >= 1; --w)
        if (L.table_bytes + (size_t)w * L.warp_bytes <= (size_t)optin) {
            L.warps = w;
            break;
        }
    if (L.warps == 0) return FSP_OK; // does not fit: the sparse walk bounds everything
    const int32_t *ptm = inst->h_ptm;
    std::vector<uint8_t> blob(L.table_bytes, 0);
    std::vector<int> order(n), A(n), B(n);
    std::vector<int32_t> S((size_t)n * (m + 1));
    for (int j = 0; j < n; ++j) {
        S[(size_t)j * (m + 1)] = 0;
        for (int i = 0; i < m; ++i) S[(size_t)j * (m + 1) + i + 1] = S[(size_t)j * (m + 1) + i] + ptm[(size_t)j * m + i];
    }
    int c = 0;
    for (int k = 0; k < m; ++k)
        for (int l = k + 1; l < m; ++l, ++c) {
            reinterpret_cast<uint32_t *>(blob.data() + L.off_kl)[c] = (uint32_t)k | ((uint32_t)l << 16);
            for (int j = 0; j < n; ++j) {
                A[j] = S[(size_t)j * (m + 1) + l] - S[(size_t)j * (m + 1) + k];
                B[j] = S[(size_t)j * (m + 1) + l + 1] - S[(size_t)j * (m + 1) + k + 1];
            }
            // Johnson-with-lags order, the same rule as the lb kernel's tables
            // (any optimal order gives the same LB, R8)
            for (int j = 0; j < n; ++j) order[j] = j;
            std::sort(order.begin(), order.end(), [&](int x, int y) {
                const bool fx = A[x] <= B[x], fy = A[y] <= B[y];
                if (fx != fy) return fx;
                if (fx ? A[x] != A[y] : B[x] != B[y]) return fx ? A[x] < A[y] : B[x] > B[y];
                return x < y;
            });
            for (int i = 0; i < n; ++i) {
                blob[L.off_pos + (size_t)c * n + order[i]] = (uint8_t)i;
                blob[L.off_jm + (size_t)c * n + i] = (uint8_t)order[i];
            }
        }
    // (p_jk, sum_{i<=k} p_ji): x = p_jl - p_jk, y = lag_j + p_jl = cum_l - cum_k
    int2 *pc = reinterpret_cast<int2 *>(blob.data() + L.off_pc);
    int *q = reinterpret_cast<int *>(blob.data() + L.off_q);
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < m; ++k) {
            pc[(size_t)j * m + k] = make_int2(ptm[(size_t)j * m + k], S[(size_t)j * (m + 1) + k + 1]);
            q[(size_t)j * m + k] = S[(size_t)j * (m + 1) + m] - S[(size_t)j * (m + 1) + k + 1];
        }
    e = cudaMalloc(&inst->d_fam, L.table_bytes);
    if (e == cudaSuccess) e = cudaMemcpy(inst->d_fam, blob.data(), L.table_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "family tables");
    inst->fam = L;
    return FSP_OK;
}

int fsp_launch_family(const fsp_instance *inst, const uint16_t *ppf, int32_t stride, const int32_t *pdp,
                      const int32_t *pC, int64_t B, const int64_t *off, const unsigned long long *ckey,
                      int32_t *out, const int *flag, cudaStream_t s)
{
    if (!inst->fam.warps) return fsp_fail(FSP_ERANGE, "family tables not available (n > 256)");
    FamArgs a;
    a.blob = inst->d_fam;
    a.L = inst->fam;
    a.n = inst->n;
    a.m = inst->m;
    a.P = inst->P;
    a.ppf = ppf;
    a.stride = stride;
    a.pdp = pdp;
    a.pC = pC;
    a.B = B;
    a.off = off;
    a.ckey = ckey;
    a.out = out;
    a.flag = flag;
    const int m = inst->m;
    if (m <= 5) return launch_family<5>(inst, a, s);
    if (m <= 10) return launch_family<10>(inst, a, s);
    if (m <= 20) return launch_family<20>(inst, a, s);
    return launch_family<32>(inst, a, s);
}

// ABI: every child of every parent with n - depth <= 32 (n <= 256).
extern "C" int fsp_lb_eval_children(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                                    const int32_t *depth, const int32_t *completion, int64_t n_parents,
                                    int32_t *lb_out, void *cuda_stream)
{
    if (!inst || n_parents < 0 || stride < 1) return fsp_fail(FSP_EINVAL, "bad arguments");
    if (n_parents == 0) return FSP_OK;
    if (!prefix || !depth || !lb_out) return fsp_fail(FSP_EINVAL, "null buffer");
    return fsp_launch_family(inst, prefix, stride, depth, completion, n_parents, nullptr, nullptr, lb_out,
                             nullptr, static_cast<cudaStream_t>(cuda_stream));
}
