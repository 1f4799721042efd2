// instance.cu — fsp_instance_load: host precompute of the per-couple tables
// (§II-D) and their one-time upload.
//
// Independent of oracle/: the couples, lags and Johnson orders are rebuilt
// here from row prefix sums, and only the two walk constants per (couple,
// position) are kept:
//   S_j[x] = sum_{i<x} p_{j,i}
//   a_j  = p_{j,k} + lag_j(k,l) = S_j[l]   - S_j[k]      (Johnson key, machine 1)
//   b_j  = lag_j(k,l) + p_{j,l} = S_j[l+1] - S_j[k+1]    (Johnson key, machine 2)
//   y_j  = b_j,   x_j  = p_{j,l} - p_{j,k}
// (the walk carries e = t2 - t1: e <- max(e + x_j, y_j))
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include "fsp_internal.h"

// Per-couple records in the layout of plan `pl` (groups, U addresses, walk form):
// [u32 (k | l<<16) x ppg][fsp_rec x np x nrec][slack] per group.
static void build_tables(const int32_t *ptm, int n, int m, const fsp_lb_plan &pl,
                         std::vector<uint8_t> &blob)
{
    // ---- couple tables, grouped: [u32 (k | l<<16) x ppg][fsp_rec x np x nrec] ----
    std::vector<int32_t> S((size_t)n * (m + 1));
    for (int j = 0; j < n; ++j) {
        S[(size_t)j * (m + 1)] = 0;
        for (int i = 0; i < m; ++i)
            S[(size_t)j * (m + 1) + i + 1] = S[(size_t)j * (m + 1) + i] + ptm[(size_t)j * m + i];
    }
    const size_t gbytes = pl.L.group_bytes;
    const size_t kl_bytes = pl.L.kl_bytes;
    // byte offset of row j of U (from the U base, lane-major rows; from the
    // warp's block, byte/nibble rows): the kernel adds the shared-window
    // address it runs at, so nothing depends on where dynamic shared memory
    // starts; row n is the always-empty padding row
    auto uaddr = [&](int j) { return (uint32_t)((size_t)j * 4 * pl.L.urow_words); };
    blob.assign(gbytes * pl.groups, 0);
    for (int g = 0; g < pl.groups; ++g) { // every record slot starts as padding
        fsp_rec *rec = reinterpret_cast<fsp_rec *>(blob.data() + (size_t)g * gbytes + kl_bytes);
        const size_t nslots = (gbytes - kl_bytes) / sizeof(fsp_rec);
        for (size_t i = 0; i < nslots; ++i) {
            rec[i].c1 = pl.s16 ? (int32_t)((uint32_t)n << 16) : 0; // job id n: never live
            rec[i].meta = pl.s16 ? (int32_t)(uaddr(n) << 16) : (int32_t)uaddr(n);
        }
    }
    std::vector<int> order(n), A(n), B(n);
    int D = 0; // 16-bit walk offset: max p (lb_kernel.cu upd<>)
    for (int64_t i = 0; i < (int64_t)n * m; ++i) D = std::max(D, (int)ptm[i]);
    int p = 0;
    for (int k = 0; k < m; ++k) {
        for (int l = k + 1; l < m; ++l, ++p) {
            const int g = p / pl.pairs_per_group, pl_idx = p % pl.pairs_per_group;
            uint8_t *gb = blob.data() + (size_t)g * gbytes;
            reinterpret_cast<uint32_t *>(gb)[pl_idx] = (uint32_t)k | ((uint32_t)l << 16);
            for (int j = 0; j < n; ++j) {
                const int32_t *Sj = &S[(size_t)j * (m + 1)];
                A[j] = Sj[l] - Sj[k];
                B[j] = Sj[l + 1] - Sj[k + 1];
            }
            // Johnson's rule on (A, B) ("with lags" P:188-190):
            // A <= B first by ascending A, then descending B; ties by job id.
            std::iota(order.begin(), order.end(), 0);
            std::sort(order.begin(), order.end(), [&](int x, int y) {
                const bool fx = A[x] <= B[x], fy = A[y] <= B[y];
                if (fx != fy) return fx;
                if (fx ? A[x] != A[y] : B[x] != B[y]) return fx ? A[x] < A[y] : B[x] > B[y];
                return x < y;
            });
            fsp_rec *rec = reinterpret_cast<fsp_rec *>(gb + kl_bytes) + (size_t)pl_idx * pl.nrec;
            if (pl.L.pos_off) // inverse position table: pos[couple][job]
                for (int i = 0; i < n; ++i) gb[pl.L.pos_off + (size_t)pl_idx * n + order[i]] = (uint8_t)i;
            for (int i = 0; i < n; ++i) {
                const int j = order[i];
                const int x = ptm[(size_t)j * m + l] - ptm[(size_t)j * m + k];
                // 16-bit walk: y + D < 2^16 in the low half, the job id in the
                // high half (read by the sparse walk's compaction only)
                rec[i].c1 = pl.s16 ? (int32_t)(((uint32_t)j << 16) | (uint32_t)(B[j] + D)) : B[j];
                rec[i].meta = pl.s16 ? (int32_t)((uaddr(j) << 16) | ((uint32_t)x & 0xffffu))
                                     : (int32_t)(((uint32_t)x << 16) | uaddr(j));
            }
        }
    }
}

// Shared-memory image of PTM for plan `pl`: int32 rows padded to mp4 (16-byte
// rows), then, TMEM plans, either the job-pair rows (pl.jp: row i, word k =
// p_{2i,k} | p_{2i+1,k} << 16, job n = 0) or the packed (p, q) machine-pair
// rows (fsp_pq_words).
static std::vector<int32_t> ptm_image(const int32_t *ptm, int n, int m, const fsp_lb_plan &pl)
{
    const int mp4 = (m + 3) & ~3;
    std::vector<int32_t> p32(pl.L.ptm_bytes / 4, 0);
    if (pl.jp) { // 16-bit (or 8-bit) rows for the C pass, then the job-pair rows
        const int w16 = fsp_ptm_row_words(true, pl.ptm8, m);
        uint32_t *p16 = reinterpret_cast<uint32_t *>(p32.data());
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < m; ++k) {
                if (pl.ptm8)
                    p16[(size_t)j * w16 + k / 4] |= (uint32_t)ptm[(size_t)j * m + k] << (8 * (k & 3));
                else
                    p16[(size_t)j * w16 + k / 2] |= (uint32_t)ptm[(size_t)j * m + k] << (16 * (k & 1));
            }
        uint32_t *jp = p16 + (((size_t)n * w16 * 4 + 15) & ~size_t(15)) / 4; // 16-byte aligned block
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < m; ++k)
                jp[(size_t)(j / 2) * mp4 + k] |= (uint32_t)ptm[(size_t)j * m + k] << (16 * (j & 1));
        return p32;
    }
    for (int j = 0; j < n; ++j)
        for (int k = 0; k < m; ++k) p32[(size_t)j * mp4 + k] = ptm[(size_t)j * m + k];
    if (pl.s16 && pl.maxm >= 10) { // nibble/TMEM variants: packed (p, q) machine pairs
        const int W = fsp_pq_words(pl.maxm), H = W / 2;
        uint32_t *pq = reinterpret_cast<uint32_t *>(p32.data() + (size_t)n * mp4);
        for (int j = 0; j < n; ++j) {
            std::vector<int32_t> pj(pl.maxm + 1, 0), qj(pl.maxm + 1, 0);
            for (int k = 0; k < m; ++k) pj[k] = ptm[(size_t)j * m + k];
            for (int l = m - 2; l >= 0; --l) qj[l] = qj[l + 1] + pj[l + 1]; // q_jl = sum_{i>l} p_ji
            for (int kp = 0; 2 * kp < m; ++kp) {
                pq[(size_t)j * W + kp] = (uint32_t)pj[2 * kp] | ((uint32_t)pj[2 * kp + 1] << 16);
                pq[(size_t)j * W + H + kp] = (uint32_t)qj[2 * kp] | ((uint32_t)qj[2 * kp + 1] << 16);
            }
        }
    }
    return p32;
}

extern "C" int fsp_instance_load(const int32_t *ptm, int32_t n, int32_t m, fsp_instance **out)
{
    if (!ptm || !out) return fsp_fail(FSP_EINVAL, "null pointer");
    *out = nullptr;
    if (n < 1 || m < 2) return fsp_fail(FSP_EINVAL, "need n >= 1 and m >= 2");
    if (n > FSP_MAX_JOBS) return fsp_fail(FSP_ERANGE, "n > FSP_MAX_JOBS");
    if (m > FSP_MAX_MACHINES) return fsp_fail(FSP_ERANGE, "m > FSP_MAX_MACHINES");
    int64_t maxp = 0;
    for (int64_t i = 0; i < (int64_t)n * m; ++i) {
        if (ptm[i] < 0) return fsp_fail(FSP_EINVAL, "negative processing time");
        maxp = std::max<int64_t>(maxp, ptm[i]);
    }
    if (maxp > 32767) return fsp_fail(FSP_ERANGE, "processing time > 32767");
    if ((int64_t)(n + m - 1) * maxp >= INT32_MAX)
        return fsp_fail(FSP_ERANGE, "(n+m-1)*max p overflows int32");

    fsp_instance *inst = new (std::nothrow) fsp_instance();
    if (!inst) return fsp_fail(FSP_ENOMEM, "host allocation");
    inst->n = n;
    inst->m = m;
    inst->P = m * (m - 1) / 2;
    inst->max_p = (int)maxp;
    cudaError_t e = cudaGetDevice(&inst->device);
    if (e != cudaSuccess) {
        delete inst;
        return fsp_cuda_fail(e, "cudaGetDevice");
    }
    inst->h_ptm = new (std::nothrow) int32_t[(size_t)n * m];
    if (!inst->h_ptm) {
        delete inst;
        return fsp_fail(FSP_ENOMEM, "host allocation");
    }
    std::memcpy(inst->h_ptm, ptm, sizeof(int32_t) * (size_t)n * m);

    int rc = fsp_plan_lb(inst, false);
    if (rc == FSP_OK) rc = fsp_plan_lb(inst, true);
    if (rc != FSP_OK) {
        fsp_instance_free(inst);
        return rc;
    }
    const fsp_lb_plan &pl = inst->plan;
    std::vector<uint8_t> blob, blob_bb;
    build_tables(ptm, n, m, inst->plan, blob);
    build_tables(ptm, n, m, inst->plan_bb, blob_bb);

    const std::vector<int32_t> p32 = ptm_image(ptm, n, m, inst->plan);
    const std::vector<int32_t> p32bb = ptm_image(ptm, n, m, inst->plan_bb);

    inst->table_bytes = (int64_t)blob.size();
    e = cudaMalloc(&inst->d_tables, blob.size());
    if (e == cudaSuccess) e = cudaMalloc(&inst->d_tables_bb, blob_bb.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(inst->d_tables_bb, blob_bb.data(), blob_bb.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&inst->d_ptm32s, pl.L.ptm_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&inst->d_ptm32s_bb, inst->plan_bb.L.ptm_bytes);
    if (e == cudaSuccess)
        e = cudaMemcpy(inst->d_ptm32s_bb, p32bb.data(), inst->plan_bb.L.ptm_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&inst->d_ptm32, sizeof(int32_t) * (size_t)n * m);
    if (e == cudaSuccess) e = cudaMalloc(&inst->d_err, sizeof(int));
    if (e == cudaSuccess)
        e = cudaMemcpy(inst->d_tables, blob.data(), blob.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(inst->d_ptm32s, p32.data(), pl.L.ptm_bytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(inst->d_ptm32, ptm, sizeof(int32_t) * (size_t)n * m, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(inst->d_err, 0, sizeof(int));
    if (e != cudaSuccess) {
        fsp_instance_free(inst);
        return fsp_cuda_fail(e, "instance upload");
    }
    rc = fsp_fam_build(inst);
    if (rc == FSP_OK && getenv("FSP_LB_MAPPING") && std::string(getenv("FSP_LB_MAPPING")) == "warp")
        rc = fsp_wpn_build(inst);
    if (rc != FSP_OK) {
        fsp_instance_free(inst);
        return rc;
    }
    *out = inst;
    return FSP_OK;
}

void fsp_host_ctx_free(void *ctx);

extern "C" void fsp_instance_free(fsp_instance *inst)
{
    if (!inst) return;
    if (inst->host_ctx) fsp_host_ctx_free(inst->host_ctx);
    if (inst->d_tables) cudaFree(inst->d_tables);
    if (inst->d_tables_bb) cudaFree(inst->d_tables_bb);
    if (inst->d_ptm32s) cudaFree(inst->d_ptm32s);
    if (inst->d_ptm32s_bb) cudaFree(inst->d_ptm32s_bb);
    if (inst->d_ptm32) cudaFree(inst->d_ptm32);
    if (inst->d_err) cudaFree(inst->d_err);
    if (inst->d_fam) cudaFree(inst->d_fam);
    if (inst->d_wpn) cudaFree(inst->d_wpn);
    delete[] inst->h_ptm;
    delete inst;
}

extern "C" int fsp_instance_get_info(const fsp_instance *inst, fsp_instance_info *info)
{
    if (!inst || !info) return fsp_fail(FSP_EINVAL, "null pointer");
    const fsp_lb_plan &pl = inst->plan;
    info->n = inst->n;
    info->m = inst->m;
    info->P = inst->P;
    info->device = inst->device;
    info->groups = pl.groups;
    info->pairs_per_group = pl.pairs_per_group;
    info->warps_per_cta = pl.warps;
    info->ctas_per_sm = pl.ctas_per_sm;
    info->smem_bytes = (int32_t)pl.smem_bytes;
    info->maxm = pl.maxm;
    info->table_bytes = inst->table_bytes;
    info->nodes_per_lane = pl.npl;
    info->walk16 = pl.s16 ? 1 : 0;
    return FSP_OK;
}

extern "C" int fsp_lb_launch_info(const fsp_instance *inst, int64_t pool, int32_t sibling,
                                  fsp_lb_launch *out)
{
    if (!inst || !out || pool < 0) return fsp_fail(FSP_EINVAL, "bad launch-info arguments");
    const fsp_lb_plan &pl = sibling ? inst->plan_bb : inst->plan;
    const int tn = 32 * pl.npl;
    const int split = fsp_lb_split(pl, pool);
    const int64_t tiles = (pool + tn - 1) / tn;
    const int64_t per_iter = (int64_t)(pl.warps / split) * pl.grid;
    out->grid = pl.grid;
    out->warps_per_cta = pl.warps;
    out->split = split;
    out->iterations = (int32_t)((tiles + per_iter - 1) / per_iter);
    out->groups = pl.groups;
    out->pairs_per_group = pl.pairs_per_group;
    out->group_buffers = pl.dbuf >= 2 ? pl.dbuf : 1;
    out->nodes_per_lane = pl.npl;
    // 0: one word per 32 nodes (lane-major), 1: a byte per lane, 2: 5-bit fields
    out->row_layout = !(pl.s16 && pl.maxm >= 10) ? 0 : pl.byte_rows ? 1 : 2;
    out->tmem_cols = pl.tm_cols;
    out->sparse_walk = pl.sparse ? 1 : 0;
    out->smem_bytes = (int32_t)pl.smem_bytes;
    out->tail_split = sibling ? 1 : fsp_lb_tail_split(pl, pool, split);
    out->heads_jp = pl.jp ? 1 : 0;
    out->mapping = !sibling && inst->wpn ? 1 : 0;
    return FSP_OK;
}
