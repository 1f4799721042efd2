/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C reference for the hot path of
 * Melab, Chakroun, Mezmaz, Tuyttens, "A GPU-accelerated Branch-and-Bound
 * Algorithm for the Flow-Shop Scheduling Problem" (arXiv 1208.3933).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1208_3933_b200/) never includes, links or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:a-b" = PAPER.md lines a-b (LaTeX source of the paper).
 * Readings of silent/garbled passages are numbered R1..Rn in DESIGN.md §3.
 *
 * All arithmetic is exact int32 (R12: LB <= (n+m-1)*max p < 2^31 is checked
 * by the caller-facing functions).
 */
#ifndef FSP_ORACLE_H
#define FSP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The six structures of §II-D / Table I, plain row-major arrays.
 *   PTM[j*m + k]     processing time of job j on machine k           (n x m)
 *   MM [2*p + 0/1]   machine couple (M1, M2) of pair index p          (P x 2)
 *   LM [j*P + p]     lag of job j on couple p                         (n x P)
 *   JM [i*P + p]     i-th job of the Johnson-with-lags order of p     (n x P)
 *   QM [j*m + l]     tail ("latency") of job j after machine l        (n x m)
 * RM (heads) depends on the node and is computed per call (Fig. 3 footnote).
 */
typedef struct {
    int32_t n, m, P;
    int32_t *PTM, *MM, *LM, *JM, *QM;
} ora_tables;

/* Table I access counters, incremented by ora_lb when non-NULL. */
typedef struct {
    int64_t jm_reads, lm_reads, ptm_reads, rm_reads, qm_reads, mm_reads;
} ora_counters;

typedef struct {
    int64_t bounded;   /* lower bounds evaluated (children)                  */
    int64_t branched;  /* nodes decomposed                                   */
    int64_t pruned;    /* children eliminated by LB >= UB                    */
    int64_t leaves;    /* complete schedules evaluated                       */
} ora_bb_stats;

/* 0 on success, -1 on bad arguments / allocation failure. */
int  ora_tables_build(const int32_t *ptm, int32_t n, int32_t m, ora_tables *t);
void ora_tables_free(ora_tables *t);

/* C_max of the (partial) sequence perm[0..len): completion time on the last
 * machine (recurrence C(i,k) = max(C(i-1,k), C(i,k-1)) + p). */
int32_t ora_makespan(const int32_t *ptm, int32_t n, int32_t m,
                     const int32_t *perm, int32_t len);

/* Johnson's two-machine rule, used for each JM column.
 * Writes the order of jobs 0..cnt-1 into order[]. */
void ora_johnson_order(const int32_t *a, const int32_t *b, int32_t cnt, int32_t *order);

/* LB of one node (prefix of length d, 0 <= d <= n), Fig. 3.
 * pair_vals (nullable, length P): timeOnM2 of each couple after line 18.
 * heads/tails (nullable, length m): the RM / QM minima the loop starts from.
 * cnt (nullable): Table I access counters (accumulated). */
int32_t ora_lb(const ora_tables *t, const uint16_t *prefix, int32_t d,
               int32_t *pair_vals, int32_t *heads, int32_t *tails, ora_counters *cnt);

/* Batched form with the fsp_lb_eval layout: node i = prefix[i*stride ..
 * i*stride + depth[i]).  Host pointers.  Returns 0, or -1 on a malformed node. */
int ora_lb_eval(const ora_tables *t, const uint16_t *prefix, int32_t stride,
                const int32_t *depth, int64_t pool, int32_t *lb_out);

/* Depth-first B&B with incumbent U = initial_ub + 1.
 * Returns 0 and the optimal makespan/permutation, 1 if no schedule has
 * makespan <= initial_ub, -1 on bad arguments. node_limit <= 0: unlimited;
 * otherwise returns 2 after node_limit bounded nodes (incumbent in *_out). */
int ora_bb_dfs(const ora_tables *t, int32_t initial_ub, int64_t node_limit,
               int32_t *makespan_out, int32_t *perm_out, ora_bb_stats *stats);

#ifdef __cplusplus
}
#endif
#endif
