// fsp_internal.h — shared declarations of libfsp.so (product path only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "fsp.h"

// Per-(couple, position) record of the pair walk, staged in shared memory.
//   c1   = y = lag_j(k,l) + p_{j,l} = sum_{k<i<=l} p_{j,i}     (int32; s16 walk:
//          low half, job id j in the high half)
//   meta = (x << 16) | addr_j   (int32 walk)  or  (addr_j << 16) | (x & 0xffff) (s16 walk)
//   x = p_{j,l} - p_{j,k} (int16); addr_j = byte offset of U row j (the kernel adds
//   its own shared-window base)
// j is the job at this position of the couple's Johnson-with-lags order.
// DESIGN.md §6 derives the one-update form e <- max(e + x, y) of Fig. 3 lines 11-15.
// Padding records after the last couple of a group (walk look-ahead).
#define FSP_REC_SLACK 8
// most couple-group buffers per CTA (multi-buffered groups)
#define FSP_MAX_GBUF 4

struct __align__(8) fsp_rec {
    int32_t c1;
    int32_t meta;
};

// u32 words per job of the packed machine-pair rows [p pairs][q pairs] that the
// nibble (TMEM) variants of the lb kernel stage after PTM: p pair = p_{j,2i} |
// p_{j,2i+1} << 16, q pair the same for the tails q_jl = sum_{i>l} p_ji; each
// half padded from ceil(maxm/2) to a multiple of 4 words.
static inline int fsp_pq_words(int maxm) { return 2 * ((((maxm + 1) / 2) + 3) & ~3); }

// u32 words per PTM row of the job-pair (jp) plans: 16-bit machine pairs
// p_{j,2i} | p_{j,2i+1} << 16, padded to 16-byte rows.
static inline int fsp_ptm16_words(int m) { return ((m + 1) / 2 + 3) & ~3; }
// ... or, when every p_jk <= 255 (fsp_lb_plan::ptm8), 8-bit rows of 8-byte
// units (one LDS.64 per 8 machines: half the C pass's gathered bytes again)
static inline int fsp_ptm8_words(int m) { return 2 * ((m + 7) / 8); }
static inline int fsp_ptm_row_words(bool jp, bool ptm8, int m)
{
    return !jp ? ((m + 3) & ~3) : ptm8 ? fsp_ptm8_words(m) : fsp_ptm16_words(m);
}

// Dynamic shared-memory layout of the lb kernel (byte offsets).
struct fsp_lb_layout {
    size_t off_u, u_bytes;     // U[(n+1)][urow_words] u32 transposed unscheduled sets (nibble
                               //   layout: one [(n+1)][urow_words] block per warp):
    int urow_words;            //   word warp*npl + q of job j's row = nodes q*32..q*32+31
    size_t off_ptm, ptm_bytes; // PTM int32 [n][mp4]
    size_t off_bar;            // mbarriers, buffer release counters, TMEM address (32 B x FSP_MAX_GBUF)
    size_t off_rt, rt_bytes;   // per warp: R, A (= R + L), Q, each [MAXM][32*npl]
    size_t off_list, list_bytes; // per warp (sparse walk): compacted records of a couple
    size_t off_tab;            // one couple group: [kl header][records]
    size_t kl_bytes, group_bytes;
    size_t pos_off;            // sparse plans, n <= 256: offset of the inverse position
                               //   table u8 [couple][job] in a group (0: none)
};

struct fsp_lb_plan {
    int maxm;            // machine-count specialisation (template)
    bool exact;          // maxm == m (5, 10, 20)
    bool s16;            // 16-bit walk (records in the s16 meta form)
    int npl;             // nodes per lane (2 or 4): U rows are 4*npl bytes per warp
    bool sparse;         // walk only the records of jobs live in the warp (B&B pools)
    int nrec;            // records per couple (n rounded up to even)
    fsp_lb_layout L;
    int groups;          // couple groups (one resident in smem at a time)
    int pairs_per_group; // couples per group (last group may be shorter)
    int dbuf;            // couple-group buffers in shared memory (0: one + CTA barrier)
    bool byte_rows;      // 16-bit walk, m >= 10: U rows of one byte per lane (else nibbles)
    bool jp;             // dense TM plans: job-pair heads (PTM + job-pair rows staged, no pq
                         //   rows; lb_kernel.cu jp_heads), jp_m = the masking offset M
    int jp_m;
    bool ptm8;           // jp plans with max p <= 255: 8-bit PTM rows for the C pass
    bool kcache;         // dense 20-machine walks: R_k, A_k cached while k is unchanged (n <= 64)
    bool recs_global;    // ablation: couple records read from global memory (20-machine dense)
    int warps;           // warps per CTA
    int ctas_per_sm;
    int num_sms;
    int smem_optin;      // cudaDevAttrMaxSharedMemoryPerBlockOptin
    int tm_cols;         // TMEM columns per CTA for the per-node R/A/Q (0: in smem)
    int grid;
    size_t smem_bytes;   // dynamic smem per CTA
};

// Shared-memory tables of the sibling-incremental (family) kernel, family.cu.
struct fsp_fam_layout {
    size_t off_kl, off_pos, off_jm, off_pc, off_q, table_bytes; // per CTA
    size_t warp_bytes;   // per-warp scratch
    int warps;           // warps per CTA (0: family kernel unavailable)
};

struct fsp_instance {
    int n, m, P;
    int device;
    int max_p;
    // host copies
    int32_t *h_ptm;
    // device tables
    uint8_t *d_tables;   // groups * group_bytes: per group [pairs][n] fsp_rec then u32 couple ids
    int32_t *d_ptm32s;   // [n][mp4] int32, padded rows + per-plan rows (lb kernel smem image, plan)
    int32_t *d_ptm32s_bb; // the same for plan_bb
    int32_t *d_ptm32;    // [n][m] int32 (B&B)
    int *d_err;          // malformed-node flag
    int64_t table_bytes;
    fsp_lb_plan plan;    // arbitrary pools (dense walk)
    fsp_lb_plan plan_bb; // B&B child pools (sparse walk, completion times supplied)
    uint8_t *d_tables_bb; // tables laid out for plan_bb
    fsp_fam_layout fam;   // family kernel tables (n <= 256)
    uint8_t *d_fam;
    // A/B (FSP_LB_MAPPING=warp at load): dense pools bounded by the warp-per-
    // sub-problem kernel of wpn.cu, records [groups][n][32] int2
    bool wpn;
    void *d_wpn;
    // host-API staging (lazily created, guarded by a mutex in api.cu)
    void *host_ctx;
};

// family kernel (family.cu): LBs of parents' children by prefix/suffix
// compositions; B&B mode (off/ckey) or every child (off == nullptr, out[p*32+t])
int fsp_fam_build(fsp_instance *inst);
int fsp_launch_family(const fsp_instance *inst, const uint16_t *ppf, int32_t stride, const int32_t *pdp,
                      const int32_t *pC, int64_t B, const int64_t *off, const unsigned long long *ckey,
                      int32_t *out, const int *flag, cudaStream_t s);

// B&B state with an explicit share of the free device memory and child
// buffer size (hybrid.cu runs several on one device)
int fsp_bb_init_ex(const fsp_instance *inst, int32_t initial_ub, int32_t rank, int32_t world,
                   double mem_frac, int64_t children_cap, bool root_only, void **state);

// warp-per-sub-problem A/B kernel (wpn.cu)
int fsp_wpn_build(fsp_instance *inst);
int fsp_launch_lb_wpn(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                      const int32_t *depth, int64_t pool, int32_t *lb_out, cudaStream_t s);

// thread-local last error
int fsp_fail(int code, const std::string &msg);
int fsp_cuda_fail(cudaError_t e, const char *what);

// lb kernel launch (lb_kernel.cu)
int fsp_plan_lb(fsp_instance *inst, bool sparse);
int fsp_lb_split(const fsp_lb_plan &pl, int64_t pool);
int fsp_lb_tail_split(const fsp_lb_plan &pl, int64_t pool, int split);
int64_t fsp_lb_tail_first(const fsp_lb_plan &pl, int64_t pool);
int fsp_launch_lb(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                  const int32_t *depth, int64_t pool, int32_t *lb_out, cudaStream_t s);
// same, pool size read on the device from *pool_dev when pool_dev != nullptr
// and, optionally, the nodes' completion times cin [pool][cin_stride] and the
// sparse-walk plan (B&B child pools)
// grid_limit > 0: at most that many CTAs (the host path leaves SMs to its
// PCIe gather kernel)
// ulist != nullptr (with cin, byte-row plans): each node's unscheduled jobs,
// n - depth entries per row; the prefix rows are then not read
int fsp_launch_lb_dev(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                      const int32_t *depth, int64_t pool, const int64_t *pool_dev,
                      const int32_t *cin, int32_t cin_stride, bool sparse, int32_t *lb_out,
                      cudaStream_t s, int grid_limit = 0, const uint16_t *ulist = nullptr);
