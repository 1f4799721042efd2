// api.cu — the bounding entry points of include/fsp.h and the error plumbing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <new>
#include <string>
#include <vector>

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
    cudaStream_t st2 = nullptr; // gather path: second bounding stream (consecutive chunks' launches overlap their tails)
    int64_t cap_nodes = 0;
    int32_t cap_stride = 0;
    uint16_t *d_pf[2] = {nullptr, nullptr};
    int32_t *d_dp[2] = {nullptr, nullptr};
    int32_t *d_lb[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};      // gather of buffer s done
    cudaEvent_t ev_done[2] = {nullptr, nullptr}; // bounding + D2H of buffer s done
};

void fsp_host_ctx_free(void *p)
{
    HostCtx *c = static_cast<HostCtx *>(p);
    if (c->st2) cudaStreamDestroy(c->st2);
    for (int s = 0; s < 2; ++s) {
        if (c->st[s]) cudaStreamDestroy(c->st[s]);
        cudaFree(c->d_pf[s]);
        cudaFree(c->d_dp[s]);
        cudaFree(c->d_lb[s]);
    }
    for (int s = 0; s < 2; ++s) {
        if (c->ev[s]) cudaEventDestroy(c->ev[s]);
        if (c->ev_done[s]) cudaEventDestroy(c->ev_done[s]);
    }
    delete c;
}

static std::mutex g_ctx_mu;

// Device address of a pinned, mapped host buffer (nullptr: pageable or not
// host memory).
template <typename T>
static T *device_view(T *p)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
    return static_cast<T *>(at.devicePointer);
}

// One warp per 8 rows in flight: depths first (lanes 0..7), then each row's
// 16-byte vectors holding prefix entries < depth (coalesced per row).
__global__ void __launch_bounds__(1024) gather_rows_kernel(const uint16_t *__restrict__ h_pf, int stride,
                                                           const int32_t *__restrict__ h_dp, int64_t cnt,
                                                           uint16_t *d_pf, int32_t *d_dp)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int s8 = stride >> 3;
    for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 8; r0 < cnt;
         r0 += warps * 8) {
        int dl = 0;
        if (lane < 8 && r0 + lane < cnt) {
            dl = h_dp[r0 + lane];
            d_dp[r0 + lane] = dl;
        }
        int d8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int du = __shfl_sync(0xffffffffu, dl, u);
            d8[u] = du > 0 ? (min(du, stride) + 7) >> 3 : 0; // a bad depth is the kernel's to flag
        }
        for (int cc = lane; cc < s8; cc += 32) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cc < d8[u]) v[u] = reinterpret_cast<const uint4 *>(h_pf + (size_t)(r0 + u) * stride)[cc];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cc < d8[u]) reinterpret_cast<uint4 *>(d_pf + (size_t)(r0 + u) * stride)[cc] = v[u];
        }
    }
}

static int eval_host_gather(const fsp_instance *inst, HostCtx *c, const uint16_t *hp, int32_t stride,
                            const int32_t *hd, int64_t pool, int32_t *lb_out)
{
    const fsp_lb_plan &pl = inst->plan;
    const int gather_sms = std::max(1, getenv("FSP_GATHER_SMS") ? atoi(getenv("FSP_GATHER_SMS")) : 8);
    const int lb_grid = std::max(1, pl.num_sms - gather_sms) * pl.ctas_per_sm;
    const int64_t tile = 32 * pl.npl;
    // chunks of one wave of tiles on the bounding SMs (no couple split); the
    // first ones are a quarter and a half wave, so the bounding starts after a
    // short gather that nothing overlaps
    const int64_t wave = (int64_t)lb_grid * pl.warps * tile;
    const int64_t chunk = std::max<int64_t>(tile, getenv("FSP_HOST_CHUNK") ? atoll(getenv("FSP_HOST_CHUNK")) : wave);
    const bool ramp = !getenv("FSP_HOST_NORAMP");
    // chunk schedule: quarter- and half-wave chunks first (the first gather
    // is not overlapped), then full waves and the remainder.  FSP_HOST_TAIL=1
    // also ends on a half and a quarter wave (the last chunk's bounding is not
    // overlapped) with the remainder after the ramp-up: measured slower at
    // 200x20 1M (8.07 vs 6.96 ms per step: the small chunks bound inefficiently)
    std::vector<int64_t> sched;
    {
        const int64_t q4 = (std::max<int64_t>(tile, chunk / 4) + tile - 1) / tile * tile;
        const int64_t q2 = (std::max<int64_t>(tile, chunk / 2) + tile - 1) / tile * tile;
        const int tail_mode = getenv("FSP_HOST_TAIL") ? atoi(getenv("FSP_HOST_TAIL")) : 0;
        const bool tail = ramp && tail_mode > 0 && pool >= 2 * (q4 + q2) + chunk;
        int64_t left = pool;
        std::vector<int64_t> head, mid, end;
        for (int64_t c : {q4, q2}) {
            if (ramp && left > 0) {
                head.push_back(std::min(c, left));
                left -= head.back();
            }
        }
        if (tail) { // 1: end on a half and a quarter wave; 2: on a half wave only
            end = tail_mode == 2 ? std::vector<int64_t>{q2} : std::vector<int64_t>{q2, q4};
            left -= tail_mode == 2 ? q2 : q2 + q4;
        }
        const int64_t full = left / chunk, rem = left - full * chunk;
        if (rem > 0 && tail) mid.push_back(rem);
        for (int64_t i = 0; i < full; ++i) mid.push_back(chunk);
        if (rem > 0 && !tail) mid.push_back(rem);
        for (auto *v : {&head, &mid, &end})
            for (int64_t c : *v) sched.push_back(c);
    }
    auto chunk_of = [&](int64_t q) { return q < (int64_t)sched.size() ? sched[q] : chunk; };
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
    if (!c->ev[0]) {
        for (int s = 0; s < 2; ++s) {
            cudaError_t e = cudaEventCreateWithFlags(&c->ev[s], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done[s], cudaEventDisableTiming);
            if (e != cudaSuccess) return fsp_cuda_fail(e, "event create");
        }
    }
    if (!c->st2) {
        cudaError_t e = cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "stream create");
    }
    // buffer s is bounded on stream lss[s]: chunk q+1's launch can start on the
    // SMs that chunk q's launch has already left (one stream would serialise
    // them, leaving every chunk's tail wave idle)
    cudaStream_t gs = c->st[1], ls = c->st[0];
    const bool two = !getenv("FSP_HOST_ONE_LB_STREAM");
    cudaStream_t lss[2] = {c->st[0], two ? c->st2 : c->st[0]};
    int64_t off = 0;
    for (int64_t q = 0; off < pool; ++q) {
        const int s = (int)(q & 1);
        const int64_t cnt = std::min(chunk_of(q), pool - off);
        cudaError_t e = cudaSuccess;
        if (q >= 2) e = cudaStreamWaitEvent(gs, c->ev_done[s], 0); // buffer s is free again
        if (e == cudaSuccess) {
            gather_rows_kernel<<<gather_sms, 1024, 0, gs>>>(hp + (size_t)off * stride, stride, hd + off, cnt,
                                                            c->d_pf[s], c->d_dp[s]);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaEventRecord(c->ev[s], gs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(lss[s], c->ev[s], 0);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "gather");
        // (FSP_GATHER_ONLY: diagnostics, the transfers without the bounding)
        // the last chunk has no gather to overlap: every SM bounds it
        const bool last = off + cnt == pool && !getenv("FSP_HOST_LASTSPLIT");
        int rc = getenv("FSP_GATHER_ONLY") ? FSP_OK
                                           : fsp_launch_lb_dev(inst, c->d_pf[s], stride, c->d_dp[s], cnt,
                                                               nullptr, nullptr, 0, false, c->d_lb[s], lss[s],
                                                               last ? 0 : lb_grid);
        if (rc != FSP_OK) return rc;
        e = cudaMemcpyAsync(lb_out + off, c->d_lb[s], sizeof(int32_t) * (size_t)cnt, cudaMemcpyDeviceToHost,
                            lss[s]);
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_done[s], lss[s]);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "D2H");
        off += cnt;
    }
    cudaError_t e = cudaStreamSynchronize(lss[0]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(lss[1]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(gs);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "sync");
    return fsp_check(inst, ls);
}

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

    // Zero-copy gather (the offload round trip of P:286-288 without the row
    // padding): when the three buffers are pinned and device-mapped, a small
    // gather kernel on a few SMs reads each node's depth and only its 2*depth
    // prefix bytes over PCIe into the device chunk buffers while the bounding
    // kernel, on the other SMs, bounds the previous chunk; LBs go back by copy.
    const uint16_t *hp = device_view(prefix);
    const int32_t *hd = device_view(depth);
    if (hp && hd && device_view(lb_out) && stride % 8 == 0 &&
        (reinterpret_cast<uintptr_t>(hp) & 15) == 0 && !getenv("FSP_HOST_COPY"))
        return eval_host_gather(inst, c, hp, stride, hd, pool, lb_out);

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

// ------------------------------------------------- runtime pool-size choice

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Synthetic D1-shaped pool on the device (DESIGN.md §5 recipe, its own
// counter-based stream): depth ~ U{0..n-1}, prefix = the first d entries of a
// random permutation (partial Fisher-Yates in the row itself).
__global__ void synth_pool_kernel(int n, int stride, int64_t N, unsigned long long seed, uint16_t *pf,
                                  int32_t *dp)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        uint16_t *row = pf + (size_t)i * stride;
        for (int j = 0; j < n; ++j) row[j] = (uint16_t)j;
        const int d = (int)(mix64(seed ^ (unsigned long long)i * 0xD1B54A32D192ED03ull) % (unsigned)n);
        for (int t = 0; t < d; ++t) {
            const unsigned long long r = mix64(seed + 0x1234567ull * (t + 1) + (unsigned long long)i * 0x9E37ull);
            const int u = t + (int)(r % (unsigned long long)(n - t));
            const uint16_t a = row[t];
            row[t] = row[u];
            row[u] = a;
        }
        dp[i] = d;
    }
}

} // namespace

// The paper sets the pool size by hand and notes it "has to be determined at
// runtime" (§VI; Table II): time the bounding kernel on
// synthetic pools of 2^12 .. 2^max_log2 nodes and return the smallest size
// whose throughput reaches `frac` of the best one.
extern "C" int fsp_lb_tune_pool(const fsp_instance *inst, int32_t max_log2, double frac, int64_t *pool_out,
                                double *rates_out, void *cuda_stream)
{
    if (!inst || !pool_out || max_log2 < 12 || max_log2 > 24 || !(frac > 0 && frac <= 1))
        return fsp_fail(FSP_EINVAL, "bad tuning arguments");
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const int n = inst->n, stride = (n + 7) & ~7;
    const int64_t Nmax = (int64_t)1 << max_log2;
    uint16_t *pf = nullptr;
    int32_t *dp = nullptr, *lb = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t e = cudaMallocAsync(&pf, sizeof(uint16_t) * (size_t)Nmax * stride, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&dp, sizeof(int32_t) * (size_t)Nmax, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&lb, sizeof(int32_t) * (size_t)Nmax, s);
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    int rc = e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "tuning buffers");
    if (rc == FSP_OK) {
        synth_pool_kernel<<<1184, 256, 0, s>>>(n, stride, Nmax, 12083933ull, pf, dp);
        e = cudaGetLastError();
        if (e != cudaSuccess) rc = fsp_cuda_fail(e, "synthetic pool");
    }
    double best = 0;
    std::vector<double> rate;
    for (int lg = 12; lg <= max_log2 && rc == FSP_OK; ++lg) {
        const int64_t N = (int64_t)1 << lg;
        const int reps = (int)std::max<int64_t>(2, std::min<int64_t>(20, ((int64_t)1 << 22) / N));
        rc = fsp_launch_lb(inst, pf, stride, dp, N, lb, s); // warm-up
        if (rc == FSP_OK) e = cudaEventRecord(e0, s);
        for (int r = 0; r < reps && rc == FSP_OK && e == cudaSuccess; ++r) rc = fsp_launch_lb(inst, pf, stride, dp, N, lb, s);
        if (rc == FSP_OK && e == cudaSuccess) e = cudaEventRecord(e1, s);
        if (rc == FSP_OK && e == cudaSuccess) e = cudaEventSynchronize(e1);
        float ms = 0;
        if (rc == FSP_OK && e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (rc == FSP_OK && e != cudaSuccess) rc = fsp_cuda_fail(e, "tuning timing");
        if (rc != FSP_OK) break;
        const double r1 = (double)N * reps / (ms * 1e-3);
        rate.push_back(r1);
        if (rates_out) rates_out[lg - 12] = r1;
        best = std::max(best, r1);
    }
    if (rc == FSP_OK) {
        *pool_out = Nmax;
        for (size_t i = 0; i < rate.size(); ++i)
            if (rate[i] >= frac * best) {
                *pool_out = (int64_t)1 << (12 + i);
                break;
            }
    }
    cudaFreeAsync(pf, s);
    cudaFreeAsync(dp, s);
    cudaFreeAsync(lb, s);
    cudaStreamSynchronize(s);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    return rc;
}
