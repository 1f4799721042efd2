/*
 * fsp.h — C ABI of libfsp.so, the B200 (sm_100a) hot path of
 * Melab, Chakroun, Mezmaz, Tuyttens, "A GPU-accelerated Branch-and-Bound
 * Algorithm for the Flow-Shop Scheduling Problem", arXiv 1208.3933.
 *
 * Citations "P:a-b" are lines of the paper's LaTeX source.
 * Readings R1..R19 of silent or garbled passages are listed in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *  - Return value: int status, FSP_OK (0) or a negative FSP_E* code; the
 *    message of the last failure on the calling thread is fsp_last_error().
 *  - "DEVICE" pointers are CUDA global-memory pointers on the device that was
 *    current when the instance was loaded (one process per GPU); "HOST"
 *    pointers are ordinary (optionally pinned) host memory.
 *  - Nothing here takes ownership of caller memory; outputs are written,
 *    inputs are only read.
 *  - cuda_stream is a cudaStream_t (NULL = legacy default stream).  Calls that
 *    take a stream are stream-ordered and asynchronous; they allocate nothing
 *    and never synchronise the host.
 */
#ifndef FSP_H
#define FSP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    FSP_OK = 0,
    FSP_EINVAL = -1,    /* null pointer, bad size, bad argument            */
    FSP_ERANGE = -2,    /* instance outside the supported value ranges     */
    FSP_ENOMEM = -3,    /* host or device allocation failed                */
    FSP_ECUDA = -4,     /* a CUDA runtime call failed                      */
    FSP_ENOTFOUND = -5, /* B&B: no schedule with makespan <= initial_ub    */
    FSP_EBUDGET = -6,   /* B&B: node/time budget exhausted before proof    */
    FSP_EBADNODE = -7   /* a malformed node was seen by a batched call     */
};

#define FSP_MAX_JOBS 4096
#define FSP_MAX_MACHINES 32

typedef struct fsp_instance fsp_instance; /* opaque, immutable after load */

/* ------------------------------------------------------------------ instance
 * fsp_instance_load — the problem statement of §II-B: n jobs,
 * m machines, processing times p_{j,k}.  Builds, on the host, the per-couple
 * structures of §II-D: the couples MM (k<l), and for
 * each couple the Johnson-with-lags order JM (R7/R8) with each
 * job's lag folded into two per-(couple, position) constants,
 * then uploads them once to the current device (the paper's "computed once
 * at the beginning").
 *   ptm     HOST, row-major [n_jobs][n_machines], ptm[j*m + k] = p_{j,k}
 *           (job-major as Fig. 3's PTM[job][M], R16).  Copied.
 *   out     receives the instance handle; free with fsp_instance_free.
 * Errors: EINVAL (null, n < 1, m < 2, any p < 0); ERANGE (n > FSP_MAX_JOBS,
 * m > FSP_MAX_MACHINES, max p > 32767, or (n+m-1)*max p >= 2^31, R12);
 * ENOMEM / ECUDA. */
int fsp_instance_load(const int32_t *ptm, int32_t n_jobs, int32_t n_machines,
                      fsp_instance **out);
void fsp_instance_free(fsp_instance *inst);

typedef struct {
    int32_t n, m, P;          /* jobs, machines, couples m(m-1)/2          */
    int32_t device;           /* CUDA ordinal the tables live on           */
    int32_t groups;           /* couple groups staged into shared memory   */
    int32_t pairs_per_group;
    int32_t warps_per_cta;    /* lb kernel launch shape                    */
    int32_t ctas_per_sm;
    int32_t smem_bytes;       /* dynamic shared memory per CTA             */
    int32_t maxm;             /* machine-count specialisation used         */
    int64_t table_bytes;      /* device bytes of the couple tables         */
    int32_t nodes_per_lane;   /* sub-problems per thread in the lb kernel  */
    int32_t walk16;           /* 1: 16-bit walk (values fit int16)         */
} fsp_instance_info;

int fsp_instance_get_info(const fsp_instance *inst, fsp_instance_info *info);

/* fsp_lb_launch_info — the launch shape fsp_lb_eval (sibling = 0) or
 * fsp_lb_eval_sibling / the B&B bounding step (sibling = 1) uses for a pool
 * of `pool` nodes (tests and bench.py report it; no device work). */
typedef struct {
    int32_t grid;             /* persistent CTAs                              */
    int32_t warps_per_cta;
    int32_t split;            /* warps sharing one 32*npl-node tile (couple split) */
    int32_t iterations;       /* tile iterations per CTA                      */
    int32_t groups;           /* couple groups cycled through shared memory   */
    int32_t pairs_per_group;
    int32_t group_buffers;    /* 1: one buffer + CTA barrier; >= 2: TMA ring  */
    int32_t nodes_per_lane;
    int32_t row_layout;       /* unscheduled-set rows: 0 word per 32 nodes,
                                 1 byte per lane, 2 5-bit fields per lane     */
    int32_t tmem_cols;        /* TMEM columns per CTA (0: heads in smem)      */
    int32_t sparse_walk;      /* 1: walk over the block's live jobs only      */
    int32_t smem_bytes;
    int32_t tail_split;       /* split of the last, partial tile iteration    */
    int32_t heads_jp;         /* 1: heads/tails/loads by job pairs (16x2 ops) */
    int32_t mapping;          /* 0: nodes over lanes (4 per lane); 1: warp per
                                 node, lanes over couples (A/B, FSP_LB_MAPPING=warp
                                 at fsp_instance_load)                         */
} fsp_lb_launch;

int fsp_lb_launch_info(const fsp_instance *inst, int64_t pool, int32_t sibling,
                       fsp_lb_launch *out);

/* ------------------------------------------------------------------- bounding
 * fsp_lb_eval — the bounding operator of §III-A applied to a pool of
 * sub-problems: lb_out[i] = LB of node i, the lower bound of
 * Fig. 3 with the readings R1-R6.
 *   prefix  DEVICE uint16 [pool][stride]; node i is the partial schedule
 *           pi(1..d) = prefix[i*stride .. i*stride + depth[i]).
 *           Entries past depth[i] are not read.  stride >= 1.
 *   depth   DEVICE int32 [pool], 0 <= depth[i] <= n.  depth == n returns the
 *           makespan (R6); depth == n-1 returns the exact makespan of the
 *           forced completion.
 *   lb_out  DEVICE int32 [pool]; fully overwritten, element i depending only
 *           on node i (order-preserving, pure).  Pools with fewer warp tiles
 *           than the GPU has warp slots are cleared first (stream-ordered
 *           memset; R1: the LB is a max from 0) and combined by atomicMax
 *           from several warps; lb_out must not alias prefix or depth.
 *   pool    number of nodes, >= 0 (0 is a no-op).
 * Malformed nodes (job >= n, repeated job, depth outside [0,n]) never cause
 * an out-of-bounds access: their LB is unspecified and a device flag is set,
 * reported as FSP_EBADNODE by fsp_check.  Errors: EINVAL, ECUDA (launch). */
int fsp_lb_eval(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                const int32_t *depth, int64_t pool, int32_t *lb_out, void *cuda_stream);

/* fsp_lb_eval_sibling — same result as fsp_lb_eval, with the sparse-walk plan
 * made for B&B child pools: when the nodes of a 64-128 node
 * block of consecutive entries share most of their unscheduled set (children
 * of nearby parents), the couple walks visit only the positions of jobs that
 * are unscheduled in at least one node of the block.
 *   completion  DEVICE int32 [pool][n_machines] or NULL: each node's prefix
 *               completion times C_k, e.g. obtained from its
 *               parent's by one step; when given, the kernel does not
 *               recompute them from the prefix (the caller guarantees they
 *               match it: a wrong C gives a wrong LB, never a fault).
 * Other arguments, layout and errors as fsp_lb_eval. */
int fsp_lb_eval_sibling(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                        const int32_t *depth, const int32_t *completion, int64_t pool,
                        int32_t *lb_out, void *cuda_stream);

/* fsp_lb_eval_children — sibling-incremental bounding (SURVEY.md §8(f)
 * NEXT-1): the LB of EVERY child of each parent (the parent's prefix + one
 * unscheduled job j, forward branching P:138-140), from one forward and one
 * backward pass per couple over the parent's unscheduled set (closed-form
 * compositions of Fig. 3's per-job updates); bit-identical to
 * fsp_lb_eval on the children.
 *   prefix, stride, depth  DEVICE parents, layout as fsp_lb_eval; every parent
 *                          must have 1 <= n - depth <= 32 (n <= 256).
 *   completion             DEVICE int32 [n_parents][n_machines] parent C_k, or
 *                          NULL (recomputed from the prefix).
 *   lb_out                 DEVICE int32 [n_parents][32]: lb_out[p*32 + t] = LB
 *                          of the child adding the t-th unscheduled job of
 *                          parent p (ascending job id), t < n - depth[p];
 *                          other entries are not written.
 * Errors: EINVAL; ERANGE (n > 256: tables not built); ECUDA. */
int fsp_lb_eval_children(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                         const int32_t *depth, const int32_t *completion, int64_t n_parents,
                         int32_t *lb_out, void *cuda_stream);

/* fsp_lb_eval_host — same result with HOST buffers (the paper's offload
 * round trip).  When prefix, depth and lb_out are pinned
 * (cudaHostAlloc / cudaHostRegister: device-mapped; stride a multiple of 8,
 * prefix 16-byte aligned), a gather kernel on 8 SMs reads each node's depth
 * and only its 2*depth prefix bytes over PCIe (zero-copy, 16-byte vectors)
 * into device chunk buffers while the bounding kernel bounds the previous
 * chunk on the other SMs; the LBs are copied back.  Otherwise whole rows are
 * copied to the device in chunks, bounded and the LBs copied back, the three
 * overlapped on two streams.  Synchronous: returns when
 * lb_out is filled.  Returns FSP_EBADNODE if a malformed node was seen.
 * Errors: EINVAL, ENOMEM, ECUDA. */
int fsp_lb_eval_host(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                     const int32_t *depth, int64_t pool, int32_t *lb_out);

/* fsp_lb_tune_pool — runtime pool-size choice (the paper: the pool size "has
 * to be determined at runtime", §VI; Table II): times
 * fsp_lb_eval on a synthetic D1-shaped pool generated on the device, for
 * pool sizes 2^12 .. 2^max_log2 (12 <= max_log2 <= 24), and returns in
 * *pool_out the smallest size whose bounds/s reach frac (0 < frac <= 1) of
 * the best.  rates_out (HOST, nullable): max_log2 - 11 doubles, bounds/s per
 * size.  Allocates (stream-ordered) and synchronises cuda_stream; not for
 * the hot path.  Errors: EINVAL, ECUDA. */
int fsp_lb_tune_pool(const fsp_instance *inst, int32_t max_log2, double frac, int64_t *pool_out,
                     double *rates_out, void *cuda_stream);

/* fsp_check — synchronises cuda_stream, then returns FSP_EBADNODE (and clears
 * the flag) if any bounding call on this instance saw a malformed node since
 * the last check, else FSP_OK. */
int fsp_check(const fsp_instance *inst, void *cuda_stream);

/* fsp_lb_work — algorithmic integer operations of Fig. 3 for one node of
 * depth d (the roofline numerator):
 *   W(d) = 2dm + n'(3m-2) + n'm + P*n + 4*P*n' + 2P,  n' = n - d. */
int64_t fsp_lb_work(int32_t n, int32_t m, int32_t d);

/* ------------------------------------------------------------------ B&B
 * fsp_bb_solve — the B&B of §II-A/§II-B with the
 * bounding, elimination and branching operators all on the device (pool never
 * round-trips through the host per iteration).  Returns a permutation with the
 * minimal makespan among those with makespan <= initial_ub
 * (INT32_MAX = unbounded); elimination prunes LB >= incumbent with the
 * incumbent started at initial_ub + 1 (R9).
 *   makespan_out  HOST int32: the optimum (or the incumbent on EBUDGET).
 *   perm_out      HOST int32 [n]: a schedule attaining it.
 *   stats         HOST, nullable.
 *   max_nodes     budget on bounded nodes (<= 0: none); time_limit_s
 *                 (<= 0: none).  On budget exhaustion returns FSP_EBUDGET
 *                 with the incumbent (not proven optimal), or FSP_ENOTFOUND
 *                 if none was found.
 * Errors: EINVAL, ENOMEM, ECUDA, ENOTFOUND, EBUDGET. */
typedef struct {
    int64_t bounded;      /* child lower bounds evaluated                  */
    int64_t branched;     /* parents decomposed                            */
    int64_t pruned;       /* children eliminated (LB >= incumbent)         */
    int64_t leaves;       /* complete schedules evaluated                  */
    int64_t iterations;   /* device expand/bound/prune steps               */
    double wall_s;        /* host wall time of the solve                   */
    int64_t lb_ops;       /* sum of fsp_lb_work over the bounded children  */
} fsp_bb_stats;

int fsp_bb_solve(const fsp_instance *inst, int32_t initial_ub, int64_t max_nodes,
                 double time_limit_s, int32_t *makespan_out, int32_t *perm_out,
                 fsp_bb_stats *stats);

/* fsp_bb_solve_hybrid — multi-core host + GPU B&B (the paper's future work,
 * P:607-609): `threads` host threads each drive their own device B&B state
 * (own stream; thread 0 starts from the root, the others empty) on the
 * current device, share the incumbent through a host
 * atomic min (adopted after every step, R9) and steal work (an idle thread's
 * request is answered with the donor's shallowest open nodes, moved device
 * to device).  Every bound, branch and elimination runs in the device
 * kernels; the host threads schedule.  Same result contract as fsp_bb_solve;
 * stats are summed over the threads.  threads in [1, 64].
 * Errors: EINVAL, ENOMEM, ECUDA, ENOTFOUND, EBUDGET. */
int fsp_bb_solve_hybrid(const fsp_instance *inst, int32_t initial_ub, int32_t threads,
                        int64_t max_nodes, double time_limit_s, int32_t *makespan_out,
                        int32_t *perm_out, fsp_bb_stats *stats);

/* Step-level B&B for the multi-GPU driver (torch.distributed owns the
 * collectives).  A state holds one device-resident pool.
 *  fsp_bb_init        state for rank/world (rank r keeps the root's
 *                     descendants assigned to it).
 *  fsp_bb_step        up to `iters` expand/bound/prune iterations.  The state
 *                     owns a stream; the iterations are ordered after work
 *                     already queued on cuda_stream, and later work on
 *                     cuda_stream after them.  Synchronous (reads the pool
 *                     size back).
 *  fsp_bb_ub_publish  writes (best << 32) | rank into a caller DEVICE int64
 *                     (stream-ordered), best = makespan of the schedule this
 *                     rank holds (INT32_MAX: none): the operand of a MIN
 *                     all-reduce, whose low 32 bits then name the holder;
 *  fsp_bb_ub_adopt    incumbent <- min(incumbent, *d_src >> 32) on the device
 *                     (after the collective); the permutation stays with the
 *                     rank in the low 32 bits of the reduced word.
 *  fsp_bb_ub_get/set  the same exchange through a HOST int64 (gloo, tests).
 *  fsp_bb_pool_size   HOST out: open nodes in the pool.
 *  fsp_bb_export      move up to max_nodes open nodes into a DEVICE buffer of
 *                     fsp_bb_node_bytes(state) bytes per node (donor side);
 *                     the buffer is complete when the call returns.
 *  fsp_bb_import      append n nodes from such a DEVICE buffer (receiver).
 *                     The copy runs on the state's stream, which is NOT
 *                     ordered after the caller's streams: the buffer's
 *                     contents must be complete before the call (e.g. after
 *                     an NCCL recv, synchronise the stream it was queued on).
 *  fsp_bb_debug_children  test hook: copy the last iteration's child pool
 *                     (every child with its LB, pruned or not) to a HOST
 *                     buffer [k][stride] u16 | [k] depth | [k][m] C | [k] LB,
 *                     stride = n rounded up to 8; *n_out = k.  max_nodes = 0:
 *                     *n_out = the number available, nothing copied.
 *  fsp_bb_result      incumbent and its permutation (HOST), FSP_ENOTFOUND if
 *                     this rank holds none.
 *  fsp_bb_get_stats   counters of this rank. */
int fsp_bb_init(const fsp_instance *inst, int32_t initial_ub, int32_t rank, int32_t world,
                void **state);
int fsp_bb_step(void *state, int32_t iters, void *cuda_stream);
int fsp_bb_ub_publish(void *state, int64_t *d_dst, void *cuda_stream);
int fsp_bb_ub_adopt(void *state, const int64_t *d_src, void *cuda_stream);
int fsp_bb_ub_get(void *state, int64_t *packed);
int fsp_bb_ub_set(void *state, int64_t packed);
int fsp_bb_pool_size(void *state, int64_t *n);
int64_t fsp_bb_node_bytes(void *state);
int fsp_bb_export(void *state, int64_t max_nodes, void *d_buf, int64_t *n_out);
int fsp_bb_import(void *state, const void *d_buf, int64_t n);
int fsp_bb_debug_children(void *state, int64_t max_nodes, void *h_buf, int64_t *n_out);
int fsp_bb_result(void *state, int32_t *makespan_out, int32_t *perm_out);
int fsp_bb_get_stats(void *state, fsp_bb_stats *stats);
void fsp_bb_free(void *state);

const char *fsp_last_error(void); /* thread-local; never NULL */
int fsp_version(void);            /* ABI version, currently 1 */

#ifdef __cplusplus
}
#endif
#endif /* FSP_H */
