// api.cu — the bounding entry points of include/fsp.h and the error plumbing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <new>
#include <string>

#include "fsp_internal.h"

static thread_local std::string g_last_error = "";

int fsp_fail(int code, const std::string &msg)
{
    g_last_error = msg;
    return code;
}

int fsp_cuda_fail(cudaError_t e, const char *what)
{
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return FSP_ECUDA;
}

extern "C" const char *fsp_last_error(void) { return g_last_error.c_str(); }

extern "C" int fsp_version(void) { return 1; }

extern "C" int64_t fsp_lb_work(int32_t n, int32_t m, int32_t d)
{
    const int64_t P = (int64_t)m * (m - 1) / 2, np = n - d;
    return 2LL * d * m + np * (3LL * m - 2) + np * m + P * n + 4LL * P * np + 2LL * P;
}

static int check_args(const fsp_instance *inst, const void *prefix, int32_t stride,
                      const void *depth, int64_t pool, const void *lb_out)
{
    if (!inst) return fsp_fail(FSP_EINVAL, "null instance");
    if (pool < 0) return fsp_fail(FSP_EINVAL, "pool < 0");
    if (pool == 0) return FSP_OK;
    if (!prefix || !depth || !lb_out) return fsp_fail(FSP_EINVAL, "null buffer");
    if (stride < 1) return fsp_fail(FSP_EINVAL, "stride < 1");
    return FSP_OK;
}

extern "C" int fsp_lb_eval(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                           const int32_t *depth, int64_t pool, int32_t *lb_out, void *cuda_stream)
{
    int rc = check_args(inst, prefix, stride, depth, pool, lb_out);
    if (rc != FSP_OK || pool == 0) return rc;
    return fsp_launch_lb(inst, prefix, stride, depth, pool, lb_out,
                         static_cast<cudaStream_t>(cuda_stream));
}

extern "C" int fsp_lb_eval_sibling(const fsp_instance *inst, const uint16_t *prefix,
                                   int32_t stride, const int32_t *depth, const int32_t *completion,
                                   int64_t pool, int32_t *lb_out, void *cuda_stream)
{
    int rc = check_args(inst, prefix, stride, depth, pool, lb_out);
    if (rc != FSP_OK || pool == 0) return rc;
    return fsp_launch_lb_dev(inst, prefix, stride, depth, pool, nullptr, completion, inst->m, true,
                             lb_out, static_cast<cudaStream_t>(cuda_stream));
}

extern "C" int fsp_check(const fsp_instance *inst, void *cuda_stream)
{
    if (!inst) return fsp_fail(FSP_EINVAL, "null instance");
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    int h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, inst->d_err, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "fsp_check");
    if (h & 2) return fsp_fail(FSP_ECUDA, "lb kernel: dynamic shared-memory base moved");
    if (h) {
        e = cudaMemsetAsync(inst->d_err, 0, sizeof(int), s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "fsp_check reset");
        return fsp_fail(FSP_EBADNODE, "malformed node in a bounded pool");
    }
    return FSP_OK;
}

// ------------------------------------------------------------ host-buffer path

struct HostCtx {
    std::mutex mu;
    cudaStream_t st[2] = {nullptr, nullptr};
    int64_t cap_nodes = 0;
    int32_t cap_stride = 0;
    uint16_t *d_pf[2] = {nullptr, nullptr};
    int32_t *d_dp[2] = {nullptr, nullptr};
    int32_t *d_lb[2] = {nullptr, nullptr};
};

void fsp_host_ctx_free(void *p)
{
    HostCtx *c = static_cast<HostCtx *>(p);
    for (int s = 0; s < 2; ++s) {
        if (c->st[s]) cudaStreamDestroy(c->st[s]);
        cudaFree(c->d_pf[s]);
        cudaFree(c->d_dp[s]);
        cudaFree(c->d_lb[s]);
    }
    delete c;
}

static std::mutex g_ctx_mu;

extern "C" int fsp_lb_eval_host(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                                const int32_t *depth, int64_t pool, int32_t *lb_out)
{
    int rc = check_args(inst, prefix, stride, depth, pool, lb_out);
    if (rc != FSP_OK || pool == 0) return rc;
    fsp_instance *mi = const_cast<fsp_instance *>(inst);
    {
        std::lock_guard<std::mutex> g(g_ctx_mu);
        if (!mi->host_ctx) {
            HostCtx *c = new (std::nothrow) HostCtx();
            if (!c) return fsp_fail(FSP_ENOMEM, "host ctx");
            for (int s = 0; s < 2; ++s) {
                cudaError_t e = cudaStreamCreateWithFlags(&c->st[s], cudaStreamNonBlocking);
                if (e != cudaSuccess) {
                    fsp_host_ctx_free(c);
                    return fsp_cuda_fail(e, "stream create");
                }
            }
            mi->host_ctx = c;
        }
    }
    HostCtx *c = static_cast<HostCtx *>(mi->host_ctx);
    std::lock_guard<std::mutex> g(c->mu);

    // chunk: about an eighth of the pool (2^16 .. 2^20 nodes, whole warp tiles),
    // so the copies of chunk i+1 overlap the kernel of chunk i and the first
    // copy, which nothing overlaps, stays short; the kernel spreads the tiles of
    // a chunk over every SM (a partial wave leaves warps idle, not SMs)
    const fsp_lb_plan &pl = inst->plan;
    const int64_t tile = 32 * pl.npl;
    int64_t chunk = std::min<int64_t>(1 << 20, std::max<int64_t>(1 << 16, (pool + 7) / 8));
    chunk = (chunk + tile - 1) / tile * tile;
    if (chunk > pool) chunk = pool;
    if (c->cap_nodes < chunk || c->cap_stride < stride) {
        for (int s = 0; s < 2; ++s) {
            cudaFree(c->d_pf[s]);
            cudaFree(c->d_dp[s]);
            cudaFree(c->d_lb[s]);
            c->d_pf[s] = nullptr;
            c->d_dp[s] = nullptr;
            c->d_lb[s] = nullptr;
        }
        c->cap_nodes = 0;
        for (int s = 0; s < 2; ++s) {
            cudaError_t e = cudaMalloc(&c->d_pf[s], sizeof(uint16_t) * (size_t)chunk * stride);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_dp[s], sizeof(int32_t) * (size_t)chunk);
            if (e == cudaSuccess) e = cudaMalloc(&c->d_lb[s], sizeof(int32_t) * (size_t)chunk);
            if (e != cudaSuccess) return fsp_cuda_fail(e, "staging allocation");
        }
        c->cap_nodes = chunk;
        c->cap_stride = stride;
    }
    int64_t nchunks = (pool + chunk - 1) / chunk;
    for (int64_t q = 0; q < nchunks; ++q) {
        const int s = (int)(q & 1);
        const int64_t off = q * chunk, cnt = std::min(chunk, pool - off);
        cudaStream_t st = c->st[s];
        cudaError_t e = cudaMemcpyAsync(c->d_pf[s], prefix + (size_t)off * stride,
                                        sizeof(uint16_t) * (size_t)cnt * stride,
                                        cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(c->d_dp[s], depth + off, sizeof(int32_t) * (size_t)cnt,
                                cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "H2D");
        rc = fsp_launch_lb(inst, c->d_pf[s], stride, c->d_dp[s], cnt, c->d_lb[s], st);
        if (rc != FSP_OK) return rc;
        e = cudaMemcpyAsync(lb_out + off, c->d_lb[s], sizeof(int32_t) * (size_t)cnt,
                            cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "D2H");
    }
    for (int s = 0; s < 2; ++s) {
        cudaError_t e = cudaStreamSynchronize(c->st[s]);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "sync");
    }
    return fsp_check(inst, c->st[0]);
}
