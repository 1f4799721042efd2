// fsp_internal.h — shared declarations of libfsp.so (product path only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "fsp.h"

// Per-(couple, position) record of the pair walk, staged in shared memory.
//   c1   = p_{j,k} + lag_j(k,l)  = sum_{k<=i<l} p_{j,i}   (int32)
//   meta = (c2 << 16) | (4*j),   c2 = p_{j,k} - p_{j,l}    (int16 in the top half)
// j is the job at this position of the couple's Johnson-with-lags order.
// DESIGN.md §6 derives the two-constant form of Fig. 3 lines 11-15.
struct __align__(8) fsp_rec {
    int32_t c1;
    int32_t meta;
};

struct fsp_lb_plan {
    int maxm;            // machine-count specialisation (template)
    int groups;          // couple groups (one resident in smem at a time)
    int pairs_per_group; // couples per group (last group may be shorter)
    int warps;           // warps per CTA
    int ctas_per_sm;
    int num_sms;
    int grid;
    size_t smem_bytes;   // dynamic smem per CTA
    size_t group_bytes;  // bytes of one group's blob (records + couple ids), 16-aligned
    size_t ptm_bytes;    // u16 PTM staged in smem, 16-aligned
    size_t warp_bytes;   // per-warp scratch
};

struct fsp_instance {
    int n, m, P;
    int device;
    int max_p;
    // host copies
    int32_t *h_ptm;
    // device tables
    uint8_t *d_tables;   // groups * group_bytes: per group [pairs][n] fsp_rec then u32 couple ids
    uint16_t *d_ptm16;   // [n][m] u16 (padded to ptm_bytes)
    int32_t *d_ptm32;    // [n][m] int32 (B&B leaf makespans)
    int *d_err;          // malformed-node flag
    int64_t table_bytes;
    fsp_lb_plan plan;
    // host-API staging (lazily created, guarded by a mutex in api.cu)
    void *host_ctx;
};

// thread-local last error
int fsp_fail(int code, const std::string &msg);
int fsp_cuda_fail(cudaError_t e, const char *what);

// lb kernel launch (lb_kernel.cu)
int fsp_plan_lb(fsp_instance *inst);
int fsp_launch_lb(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                  const int32_t *depth, int64_t pool, int32_t *lb_out, cudaStream_t s);
