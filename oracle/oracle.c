/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path of
 * arXiv 1208.3933 computes, written in the paper's order and notation:
 *
 *   - the six structures PTM, LM, JM, RM, QM, MM of §II-D (Table I
 *     P:206-232), built by ora_tables_build;
 *   - the lower bound LB of Fig. 3, ora_lb, line by line;
 *   - a depth-first B&B with the four operators of §II-A and the
 *     forward branching of §II-B, ora_bb_dfs.
 *
 * Readings of passages the paper leaves silent or garbled are cited as R1..R19
 * (taken from SURVEY.md §8(c) A1..A18).  No blocking, fusion or
 * reordering beyond what Fig. 3 states.  Nothing here is shared with the CUDA
 * path.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

static int32_t imax(int32_t a, int32_t b) { return a > b ? a : b; }
static int32_t imin(int32_t a, int32_t b) { return a < b ? a : b; }

/* ---------------------------------------------------------------- makespan */

/* P:158-160 "the makespan C_max, which represents the completion time of the
 * last scheduled job on the last machine"; permutation FSP:
 *   C(i,k) = max(C(i-1,k), C(i,k-1)) + p_{perm(i),k},  C(0,.) = C(.,0) = 0. */
int32_t ora_makespan(const int32_t *ptm, int32_t n, int32_t m,
                     const int32_t *perm, int32_t len)
{
    (void)n;
    int32_t *C = (int32_t *)calloc((size_t)m, sizeof(int32_t));
    for (int32_t i = 0; i < len; ++i) {
        int32_t prev = 0; /* C(i, k-1) */
        for (int32_t k = 0; k < m; ++k) {
            C[k] = imax(C[k], prev) + ptm[perm[i] * m + k];
            prev = C[k];
        }
    }
    int32_t cmax = len > 0 ? C[m - 1] : 0;
    free(C);
    return cmax;
}

/* ----------------------------------------------------------- Johnson's rule */

/* Johnson's algorithm for two machines ([SMJohnson_54]): jobs with
 * a_j <= b_j first in non-decreasing a_j, then jobs with a_j > b_j in
 * non-increasing b_j; ties by ascending job id (R8).  Plain insertion sort. */
static int johnson_before(const int32_t *a, const int32_t *b, int32_t x, int32_t y)
{
    int sx = a[x] <= b[x] ? 0 : 1, sy = a[y] <= b[y] ? 0 : 1;
    if (sx != sy) return sx < sy;
    if (sx == 0) { if (a[x] != a[y]) return a[x] < a[y]; }
    else         { if (b[x] != b[y]) return b[x] > b[y]; }
    return x < y;
}

void ora_johnson_order(const int32_t *a, const int32_t *b, int32_t cnt, int32_t *order)
{
    for (int32_t i = 0; i < cnt; ++i) {
        int32_t j = i;
        while (j > 0 && johnson_before(a, b, i, order[j - 1])) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = i;
    }
}

/* ------------------------------------------------------------ the tables */

int ora_tables_build(const int32_t *ptm, int32_t n, int32_t m, ora_tables *t)
{
    if (!ptm || !t || n < 1 || m < 2) return -1;
    memset(t, 0, sizeof(*t));
    t->n = n;
    t->m = m;
    t->P = m * (m - 1) / 2; /* couples (M_k, M_l), k < l */
    int32_t P = t->P;
    t->PTM = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * m);
    t->MM = (int32_t *)malloc(sizeof(int32_t) * (size_t)P * 2);
    t->LM = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * P);
    t->JM = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * P);
    t->QM = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * m);
    if (!t->PTM || !t->MM || !t->LM || !t->JM || !t->QM) { ora_tables_free(t); return -1; }

    /* PTM: "the processing times of all the jobs on all the machines"
     * (P:198-200), indexed PTM[job][M] as in Fig. 3 lines 11-15 (R16). */
    int64_t maxp = 0;
    for (int32_t j = 0; j < n * m; ++j) {
        if (ptm[j] < 0) { ora_tables_free(t); return -1; }
        t->PTM[j] = ptm[j];
        if (ptm[j] > maxp) maxp = ptm[j];
    }
    /* R12: every quantity is at most (n+m-1)*max p; keep it inside int32. */
    if ((int64_t)(n + m - 1) * maxp >= INT32_MAX) { ora_tables_free(t); return -1; }

    /* MM: "the matrix MM containing the couples of machines", each
     * couple (M_k, M_l) with k < l, lexicographic (R15). */
    int32_t p = 0;
    for (int32_t k = 0; k < m; ++k)
        for (int32_t l = k + 1; l < m; ++l) {
            t->MM[2 * p + 0] = k;
            t->MM[2 * p + 1] = l;
            ++p;
        }

    /* LM: "the lag of each remaining job ... on the couple (M_k, M_l)"
     * computed once: lag_j(k,l) = sum of p_ji for k < i < l. */
    for (int32_t j = 0; j < n; ++j)
        for (p = 0; p < P; ++p) {
            int32_t k = t->MM[2 * p], l = t->MM[2 * p + 1], lag = 0;
            for (int32_t i = k + 1; i < l; ++i) lag += t->PTM[j * m + i];
            t->LM[j * P + p] = lag;
        }

    /* JM: per couple, "Johnson's rule with lags" (R7): Johnson's
     * order on the virtual two-machine times (p_jk + lag_j, lag_j + p_jl). */
    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *b = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (p = 0; p < P; ++p) {
        int32_t k = t->MM[2 * p], l = t->MM[2 * p + 1];
        for (int32_t j = 0; j < n; ++j) {
            a[j] = t->PTM[j * m + k] + t->LM[j * P + p];
            b[j] = t->LM[j * P + p] + t->PTM[j * m + l];
        }
        ora_johnson_order(a, b, n, order);
        for (int32_t i = 0; i < n; ++i) t->JM[i * P + p] = order[i];
    }
    free(a);
    free(b);
    free(order);

    /* QM: "lowest latency times", per job the work remaining after
     * machine l: q_jl = sum of p_ji for i > l (R4). */
    for (int32_t j = 0; j < n; ++j)
        for (int32_t l = 0; l < m; ++l) {
            int32_t q = 0;
            for (int32_t i = l + 1; i < m; ++i) q += t->PTM[j * m + i];
            t->QM[j * m + l] = q;
        }
    return 0;
}

void ora_tables_free(ora_tables *t)
{
    if (!t) return;
    free(t->PTM); free(t->MM); free(t->LM); free(t->JM); free(t->QM);
    memset(t, 0, sizeof(*t));
}

/* ------------------------------------------------------------- the bound */

/* LB of the sub-problem pi(1..d), following Fig. 3. */
int32_t ora_lb(const ora_tables *t, const uint16_t *prefix, int32_t d,
               int32_t *pair_vals, int32_t *heads, int32_t *tails, ora_counters *cnt)
{
    const int32_t n = t->n, m = t->m, P = t->P;
    const int32_t *PTM = t->PTM, *MM = t->MM, *LM = t->LM, *JM = t->JM, *QM = t->QM;

    /* "job not yet scheduled" (Fig. 3 line 10): the jobs of pi(1..d). */
    char *scheduled = (char *)calloc((size_t)n, 1);
    for (int32_t i = 0; i < d; ++i) scheduled[prefix[i]] = 1;

    /* Completion times of the partial schedule on each machine,
     * the permutation-FSP recurrence over pi(1..d). */
    int32_t *C = (int32_t *)calloc((size_t)m, sizeof(int32_t));
    for (int32_t i = 0; i < d; ++i) {
        int32_t prev = 0;
        for (int32_t k = 0; k < m; ++k) {
            C[k] = imax(C[k], prev) + PTM[prefix[i] * m + k];
            prev = C[k];
        }
    }

    /* R6: a complete schedule (d == n) bounds to its own makespan. */
    if (d == n) {
        int32_t cmax = C[m - 1];
        if (heads) for (int32_t k = 0; k < m; ++k) heads[k] = C[k];
        if (tails) for (int32_t k = 0; k < m; ++k) tails[k] = 0;
        if (pair_vals) for (int32_t p = 0; p < P; ++p) pair_vals[p] = C[MM[2 * p + 1]];
        free(scheduled);
        free(C);
        return cmax;
    }

    /* RM: "earliest starting times of jobs", per unscheduled job j
     * (R3): r_j0 = C_0, r_jk = max(C_k, r_j,k-1 + p_j,k-1).  Fig. 3 lines
     * 06-07 take min over the jobs (footnote P:242: minima computed on the
     * CPU); the minimum ranges over unscheduled jobs only (R5). */
    int32_t *RMmin = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    int32_t *QMmin = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    int32_t *r = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    for (int32_t k = 0; k < m; ++k) { RMmin[k] = INT32_MAX; QMmin[k] = INT32_MAX; }
    for (int32_t j = 0; j < n; ++j) {
        if (scheduled[j]) continue;
        r[0] = C[0];
        for (int32_t k = 1; k < m; ++k) r[k] = imax(C[k], r[k - 1] + PTM[j * m + k - 1]);
        for (int32_t k = 0; k < m; ++k) {
            RMmin[k] = imin(RMmin[k], r[k]);
            /* Fig. 3 line 18: min over jobs of QM[M2][j] (R4, R5). */
            QMmin[k] = imin(QMmin[k], QM[j * m + k]);
        }
    }
    if (heads) for (int32_t k = 0; k < m; ++k) heads[k] = RMmin[k];
    if (tails) for (int32_t k = 0; k < m; ++k) tails[k] = QMmin[k];

    int32_t LB = 0; /* line 02, R1: a max over couples starts at 0 */
    for (int32_t index = 0; index < P; ++index) {                   /* 03 */
        int32_t M1 = MM[2 * index + 0];                              /* 04 */
        int32_t M2 = MM[2 * index + 1];                              /* 05 */
        int32_t timeOnM1 = RMmin[M1];                                /* 06 */
        int32_t timeOnM2 = RMmin[M2];                                /* 07 */
        if (cnt) { cnt->mm_reads += 2; cnt->rm_reads += 2; }
        for (int32_t i = 0; i < n; ++i) {                            /* 08 */
            int32_t job = JM[i * P + index];                         /* 09 */
            if (cnt) cnt->jm_reads += 1;
            if (!scheduled[job]) {                                   /* 10 */
                timeOnM1 = timeOnM1 + PTM[job * m + M1];             /* 11 */
                int32_t lag = LM[job * P + index];
                if (cnt) { cnt->ptm_reads += 2; cnt->lm_reads += 1; }
                if (timeOnM2 > timeOnM1 + lag)                       /* 12 */
                    timeOnM2 += PTM[job * m + M2];                   /* 13 */
                else                                                 /* 14 */
                    timeOnM2 = timeOnM1 + lag + PTM[job * m + M2];   /* 15 */
            }                                                        /* 16 */
        }                                                            /* 17 */
        timeOnM2 += QMmin[M2];                                       /* 18 */
        if (cnt) cnt->qm_reads += 1;
        if (pair_vals) pair_vals[index] = timeOnM2;
        LB = imax(timeOnM2, LB);                                     /* 19 */
    }                                                                /* 20 */
    free(scheduled);
    free(C);
    free(RMmin);
    free(QMmin);
    free(r);
    return LB;                                                       /* 21 */
}

/* Pool of sub-problems evaluated one by one (the serial counterpart of the
 * pool offload of §III-A).  Node validity is checked (R6/API). */
int ora_lb_eval(const ora_tables *t, const uint16_t *prefix, int32_t stride,
                const int32_t *depth, int64_t pool, int32_t *lb_out)
{
    char *seen = (char *)malloc((size_t)t->n);
    int rc = 0;
    for (int64_t i = 0; i < pool; ++i) {
        const uint16_t *pf = prefix + (size_t)i * (size_t)stride;
        int32_t d = depth[i];
        if (d < 0 || d > t->n || d > stride) { rc = -1; lb_out[i] = -1; continue; }
        memset(seen, 0, (size_t)t->n);
        int bad = 0;
        for (int32_t q = 0; q < d; ++q) {
            if (pf[q] >= t->n || seen[pf[q]]) { bad = 1; break; }
            seen[pf[q]] = 1;
        }
        if (bad) { rc = -1; lb_out[i] = -1; continue; }
        lb_out[i] = ora_lb(t, pf, d, NULL, NULL, NULL, NULL);
    }
    free(seen);
    return rc;
}

/* -------------------------------------------------------------- the B&B */

typedef struct {
    const ora_tables *t;
    int32_t U;            /* incumbent + the strict-prune convention (R9) */
    int have;             /* a schedule has been stored                   */
    int32_t *best;        /* best permutation found                       */
    uint16_t *prefix;     /* current partial schedule                     */
    char *scheduled;
    int64_t limit;
    int stopped;
    ora_bb_stats st;
} dfs_ctx;

typedef struct { int32_t lb, idle, job; } kid;

/* Best-first order among sons (R10): ascending LB; equal LBs by ascending
 * idle time the son's job adds (R19), then by job id. */
static int kid_cmp(const void *x, const void *y)
{
    const kid *a = (const kid *)x, *b = (const kid *)y;
    if (a->lb != b->lb) return a->lb < b->lb ? -1 : 1;
    if (a->idle != b->idle) return a->idle < b->idle ? -1 : 1;
    return a->job < b->job ? -1 : (a->job > b->job);
}

/* Completion times C[k] of the prefix on every machine (the
 * recurrence of ora_makespan kept per machine). */
static void prefix_completion(const ora_tables *t, const uint16_t *prefix, int32_t d, int32_t *C)
{
    for (int32_t k = 0; k < t->m; ++k) C[k] = 0;
    for (int32_t i = 0; i < d; ++i) {
        int32_t prev = 0;
        for (int32_t k = 0; k < t->m; ++k) {
            C[k] = imax(C[k], prev) + t->PTM[prefix[i] * t->m + k];
            prev = C[k];
        }
    }
}

/* R19: idle time appending job j adds: machine k, free at C[k], waits until
 * j leaves machine k-1; sum over k of (start of j on k) - C[k]. */
static int32_t son_idle(const ora_tables *t, const int32_t *C, int32_t j)
{
    int32_t idle = 0, prev = 0;
    for (int32_t k = 0; k < t->m; ++k) {
        const int32_t start = imax(C[k], prev);
        idle += start - C[k];
        prev = start + t->PTM[j * t->m + k];
    }
    return idle;
}

/* Store a complete schedule (prefix[0..n)) if it improves on U. */
static void leaf(dfs_ctx *c)
{
    const ora_tables *t = c->t;
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)t->n);
    for (int32_t i = 0; i < t->n; ++i) perm[i] = c->prefix[i];
    int32_t cmax = ora_makespan(t->PTM, t->n, t->m, perm, t->n);
    c->st.leaves++;
    if (cmax < c->U) {
        c->U = cmax;
        c->have = 1;
        memcpy(c->best, perm, sizeof(int32_t) * (size_t)t->n);
    }
    free(perm);
}

/* Decompose the node prefix[0..d) (branching: son i schedules job
 * J_i next), bound every son (Fig. 3), eliminate sons with LB >= U (R9),
 * and explore the rest depth-first in ascending (LB, idle, job) order (R10,
 * R19). */
static void dfs(dfs_ctx *c, int32_t d)
{
    const ora_tables *t = c->t;
    const int32_t n = t->n;
    if (c->stopped) return;
    c->st.branched++;
    if (d == n - 1) { /* one son: its schedule is complete */
        for (int32_t j = 0; j < n; ++j)
            if (!c->scheduled[j]) c->prefix[d] = (uint16_t)j;
        leaf(c);
        return;
    }
    kid *kids = (kid *)malloc(sizeof(kid) * (size_t)n);
    int32_t *C = (int32_t *)malloc(sizeof(int32_t) * (size_t)t->m);
    prefix_completion(t, c->prefix, d, C);
    int32_t nk = 0;
    for (int32_t j = 0; j < n; ++j) {
        if (c->scheduled[j]) continue;
        c->prefix[d] = (uint16_t)j;
        if (d + 1 == n - 1) {
            /* the son's only completion: evaluate it as a schedule */
            c->scheduled[j] = 1;
            for (int32_t q = 0; q < n; ++q)
                if (!c->scheduled[q]) c->prefix[d + 1] = (uint16_t)q;
            c->scheduled[j] = 0;
            leaf(c);
            continue;
        }
        int32_t lb = ora_lb(t, c->prefix, d + 1, NULL, NULL, NULL, NULL);
        c->st.bounded++;
        if (lb >= c->U) { c->st.pruned++; continue; }
        kids[nk].lb = lb;
        kids[nk].idle = son_idle(t, C, j);
        kids[nk].job = j;
        ++nk;
    }
    if (c->limit > 0 && c->st.bounded >= c->limit) c->stopped = 1;
    qsort(kids, (size_t)nk, sizeof(kid), kid_cmp);
    for (int32_t q = 0; q < nk && !c->stopped; ++q) {
        if (kids[q].lb >= c->U) { c->st.pruned++; continue; }
        c->prefix[d] = (uint16_t)kids[q].job;
        c->scheduled[kids[q].job] = 1;
        dfs(c, d + 1);
        c->scheduled[kids[q].job] = 0;
    }
    free(kids);
    free(C);
}

int ora_bb_dfs(const ora_tables *t, int32_t initial_ub, int64_t node_limit,
               int32_t *makespan_out, int32_t *perm_out, ora_bb_stats *stats)
{
    if (!t || !makespan_out || !perm_out || initial_ub < 0) return -1;
    dfs_ctx c;
    memset(&c, 0, sizeof(c));
    c.t = t;
    c.U = initial_ub == INT32_MAX ? INT32_MAX : initial_ub + 1; /* R9 */
    c.best = (int32_t *)malloc(sizeof(int32_t) * (size_t)t->n);
    c.prefix = (uint16_t *)calloc((size_t)t->n + 1, sizeof(uint16_t));
    c.scheduled = (char *)calloc((size_t)t->n, 1);
    c.limit = node_limit;
    dfs(&c, 0);
    int rc = c.stopped ? 2 : (c.have ? 0 : 1);
    *makespan_out = c.have ? c.U : -1;
    if (c.have) memcpy(perm_out, c.best, sizeof(int32_t) * (size_t)t->n);
    if (stats) *stats = c.st;
    free(c.best);
    free(c.prefix);
    free(c.scheduled);
    return rc;
}
