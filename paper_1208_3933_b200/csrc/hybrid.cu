// hybrid.cu — multi-core host + GPU B&B (the paper's
// future work P:607-609): T host threads, each driving its own device B&B
// state (its own stream, its share of the root's children) on the
// same GPU, so several selection/branching fronts keep the device busy where
// one front's iterations are small or wait on their host round trip.  Thread
// 0 starts from the root (its first dive keeps the best-first order of the
// root's children, R19); the others start empty and steal.
//   * incumbent: a host atomic min of the packed (makespan << 32 | thread)
//     words, adopted by every state after each of its steps (R9 pruning);
//   * work stealing: an idle thread posts a request, a thread with a large
//     pool exports its shallowest open nodes (largest subtrees) into a device
//     buffer that the idle thread imports (device-to-device copies);
//   * termination: every thread idle with no transfer in flight.
// All bounding, branching and elimination run in the device kernels of
// lb_kernel.cu / bb.cu; the host threads only select when to step, share the
// incumbent and move open nodes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "fsp_internal.h"

namespace {

struct Transfer {
    void *buf;
    int64_t k;
};

struct Shared {
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Transfer> ready; // exported node buffers waiting for an idle thread
    int idle = 0;               // threads with an empty pool, waiting
    int requests = 0;           // unanswered requests for work
    bool done = false;
    int rc = FSP_OK;
    std::atomic<long long> best{((long long)INT32_MAX << 32)};
    std::atomic<bool> stop{false};
};

void worker(const fsp_instance *inst, void *st, int tid, int T, Shared &sh, int iters_per_step,
            int64_t node_bytes, std::atomic<long long> &bounded_total, int64_t max_nodes,
            std::chrono::steady_clock::time_point t_end, bool timed)
{
    cudaSetDevice(inst->device);
    auto fail = [&](int rc) {
        std::lock_guard<std::mutex> g(sh.mu);
        if (sh.rc == FSP_OK) sh.rc = rc;
        sh.done = true;
        sh.stop = true;
        sh.cv.notify_all();
    };
    long long last_bounded = 0;
    for (;;) {
        if (sh.stop.load()) return;
        int64_t open = 0;
        int rc = fsp_bb_pool_size(st, &open);
        if (rc == FSP_OK && open > 0) {
            rc = fsp_bb_step(st, iters_per_step, nullptr);
            if (rc != FSP_OK) return fail(rc);
            // incumbent: publish this thread's best, adopt the global one
            long long mine = 0;
            rc = fsp_bb_ub_get(st, reinterpret_cast<int64_t *>(&mine));
            if (rc != FSP_OK) return fail(rc);
            long long cur = sh.best.load();
            while (mine < cur && !sh.best.compare_exchange_weak(cur, mine)) {
            }
            rc = fsp_bb_ub_set(st, sh.best.load());
            if (rc != FSP_OK) return fail(rc);
            fsp_bb_stats bs;
            rc = fsp_bb_get_stats(st, &bs);
            if (rc != FSP_OK) return fail(rc);
            bounded_total += bs.bounded - last_bounded;
            last_bounded = bs.bounded;
            if ((max_nodes > 0 && bounded_total.load() >= max_nodes) ||
                (timed && std::chrono::steady_clock::now() >= t_end)) {
                std::lock_guard<std::mutex> g(sh.mu);
                sh.stop = true;
                sh.cv.notify_all();
                return;
            }
            // donate to an idle thread: half the pool (at most 64K nodes)
            rc = fsp_bb_pool_size(st, &open);
            if (rc != FSP_OK) return fail(rc);
            bool give = false;
            {
                std::lock_guard<std::mutex> g(sh.mu);
                if (sh.requests > 0 && open >= 64) {
                    --sh.requests;
                    give = true;
                }
            }
            if (give) {
                const int64_t k = std::min<int64_t>(open / 2, 1 << 16);
                void *buf = nullptr;
                cudaError_t e = cudaMalloc(&buf, (size_t)k * node_bytes);
                if (e != cudaSuccess) return fail(fsp_cuda_fail(e, "hybrid transfer buffer"));
                int64_t got = 0;
                rc = fsp_bb_export(st, k, buf, &got); // synchronous: buf complete on return
                if (rc != FSP_OK) return fail(rc);
                std::lock_guard<std::mutex> g(sh.mu);
                sh.ready.push_back({buf, got});
                sh.cv.notify_all();
            }
            continue;
        }
        if (rc != FSP_OK) return fail(rc);
        // empty pool: ask for work; done when every thread is idle
        Transfer tr{nullptr, 0};
        {
            std::unique_lock<std::mutex> g(sh.mu);
            ++sh.idle;
            ++sh.requests;
            for (;;) {
                if (sh.done || sh.stop) {
                    --sh.idle;
                    return;
                }
                if (!sh.ready.empty()) {
                    tr = sh.ready.front();
                    sh.ready.pop_front();
                    break;
                }
                if (sh.idle == T) { // nobody works and nothing is in flight
                    sh.done = true;
                    sh.cv.notify_all();
                    --sh.idle;
                    return;
                }
                sh.cv.wait(g);
            }
            --sh.idle;
        }
        if (tr.k > 0) {
            rc = fsp_bb_import(st, tr.buf, tr.k);
            cudaFree(tr.buf);
            if (rc != FSP_OK) return fail(rc);
        } else {
            cudaFree(tr.buf);
        }
    }
}

} // namespace

extern "C" int fsp_bb_solve_hybrid(const fsp_instance *inst, int32_t initial_ub, int32_t threads,
                                   int64_t max_nodes, double time_limit_s, int32_t *makespan_out,
                                   int32_t *perm_out, fsp_bb_stats *stats)
{
    if (!inst || !makespan_out || !perm_out || threads < 1 || threads > 64 || initial_ub < 0)
        return fsp_fail(FSP_EINVAL, "bad hybrid B&B arguments");
    const auto t0 = std::chrono::steady_clock::now();
    const int T = threads;
    std::vector<void *> st(T, nullptr);
    int rc = FSP_OK;
    for (int t = 0; t < T && rc == FSP_OK; ++t)
        rc = fsp_bb_init_ex(inst, initial_ub, t, T, 0.5 / T, (int64_t)(1 << 21) / T, true, &st[t]);
    if (rc != FSP_OK) {
        for (void *s : st) fsp_bb_free(s);
        return rc;
    }
    Shared sh;
    std::atomic<long long> bounded_total{0};
    const bool timed = time_limit_s > 0;
    const auto t_end = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                                 std::chrono::duration<double>(timed ? time_limit_s : 0.0));
    const int64_t nb = fsp_bb_node_bytes(st[0]);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back(worker, inst, st[t], t, T, std::ref(sh), 4, nb, std::ref(bounded_total), max_nodes,
                        t_end, timed);
    for (auto &x : th) x.join();
    for (const Transfer &tr : sh.ready) cudaFree(tr.buf);
    rc = sh.rc;
    const bool budget = sh.stop.load() && rc == FSP_OK;
    // the winner: the state whose schedule has the smallest makespan
    fsp_bb_stats tot{};
    int32_t best = -1;
    int winner = -1;
    for (int t = 0; t < T && rc == FSP_OK; ++t) {
        fsp_bb_stats s1;
        rc = fsp_bb_get_stats(st[t], &s1);
        tot.bounded += s1.bounded;
        tot.branched += s1.branched;
        tot.pruned += s1.pruned;
        tot.leaves += s1.leaves;
        tot.iterations += s1.iterations;
        tot.lb_ops += s1.lb_ops;
        int32_t ms = -1;
        std::vector<int32_t> p(inst->n);
        const int r1 = fsp_bb_result(st[t], &ms, p.data());
        if (r1 == FSP_OK && (winner < 0 || ms < best)) {
            best = ms;
            winner = t;
            std::copy(p.begin(), p.end(), perm_out);
        }
    }
    tot.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats) *stats = tot;
    for (void *s : st) fsp_bb_free(s);
    if (rc != FSP_OK) return rc;
    *makespan_out = best;
    if (budget) return fsp_fail(winner >= 0 ? FSP_EBUDGET : FSP_ENOTFOUND, "B&B budget exhausted");
    return winner >= 0 ? FSP_OK : fsp_fail(FSP_ENOTFOUND, "no schedule within the upper bound");
}
