// lb_kernel.cu — batched Lageweg-Lenstra-Rinnooy Kan two-machine bound on sm_100a.
//
// Computes, for every node of a pool, the LB of Fig. 3 with the
// readings R1-R6 of DESIGN.md §3.  Design:
//   * one thread per sub-problem, as the paper maps it — here four
//     sub-problems per thread (two for generic m), 128 per warp, so every table
//     read of the couple walk is warp-uniform (a shared-memory broadcast);
//   * the per-couple tables (Johnson-with-lags order with each job's constants
//     folded into an 8-byte record) are staged into shared memory by TMA bulk
//     copies (cp.async.bulk + mbarrier), in couple groups held in two buffers
//     when the whole set exceeds shared memory (200x20: 8 groups of 24);
//   * the unscheduled sets of a warp's nodes are a transposed bitset, one row
//     per job: a byte per lane (16-bit walk, m >= 10), 5-bit fields (long job
//     lists) or one word per 32 nodes (m = 5, int32 walk); each record carries
//     the row's offset, so one multiply-add addresses a lane's mask;
//   * per-node heads/tails (R, A = R + L, Q) live in tensor memory (TMEM);
//   * phase A (completion times C_k, heads, tails, loads; rows a1-a3): the
//     tile's nodes are dealt to the slots by depth rank (a warp bitonic sort),
//     C_k comes from a 16-bit (5 machines: 8-bit) PTM-row pass that also sums
//     the loads, the heads and tails run over job PAIRS in 16x2 ops with
//     scheduled halves pushed above every real value (jp_heads, no branch);
//   * the walk of Fig. 3 lines 08-17 is carried in the difference form
//     e = timeOnM2 - timeOnM1:
//         e <- max(e + x_j, y_j)      (if j unscheduled)
//     x_j = p_jl - p_jk, y_j = lag_j + p_jl: one predicated VIADDMNMX per
//     update, exact integer arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <string>
#include <cstdlib>
#include <type_traits>

#include "fsp_internal.h"


// node data read once per launch (depths, prefixes) as streaming loads
// (evict-first), meant to keep the TMA ring's records in L2: measured off
// (profiles/r02/stream_loads_ab.txt: DRAM reads 336 -> 384 MB per 200x20
// launch, same time), so plain loads
#ifndef FSP_STREAM_LOADS
#define FSP_STREAM_LOADS 0
#endif
#if FSP_STREAM_LOADS
#define FSP_LDS_STREAM(p) __ldcs(p)
#else
#define FSP_LDS_STREAM(p) (*(p))
#endif
// job-pair heads: two pairs per loop iteration (VIMNMX3 folds); FSP_JP_SPLIT:
// the tails in a second pass over the pairs
#ifndef FSP_JP2
#define FSP_JP2 1
#endif
#ifndef FSP_JP_SPLIT
#define FSP_JP_SPLIT 0
#endif
// job-pair heads: byte-row flags by one PRMT (A/B switch)
#ifndef FSP_JP_BYTEFLAGS
#define FSP_JP_BYTEFLAGS 0 // measured: no difference (profiles/r02/jp_byteflags_ab.txt)
#endif
// job-pair heads take the loads from the C pass (L = total - prefix sums)
#ifndef FSP_JP_LC
#define FSP_JP_LC 1
#endif
// walk-loop unroll (x two 4-position steps per iteration), measured per
// variant (profiles/r02/walk_unroll_ab.txt): 200x20 (dense, long lists) 8,
// KC (n <= 64) 4, 5 machines 1; sparse (B&B) walks FSP_WALK_UNROLL_SPARSE
#ifndef FSP_WALK_UNROLL_SPARSE
#define FSP_WALK_UNROLL_SPARSE 1
#endif
#ifndef FSP_WALK_UNROLL_DENSE
#define FSP_WALK_UNROLL_DENSE 8
#endif

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// The waiting warp suspends in try_wait (time hint) instead of spinning: a
// spin loop here took 9 % of the issue slots of the walk's SM (ncu v12).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, uint32_t hint_ns = 1000000u)
{
    uint32_t done = 0;
    while (!done) {
        if (hint_ns) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
                : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_u32(bar)), "r"(parity)
                : "memory");
        }
    }
}

// TMA 1-D bulk copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Issue the bulk copies of `bytes` (multiple of 16) in <= 32 KB pieces.
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    const uint32_t piece = 32768;
    for (uint32_t off = 0; off < bytes; off += piece) {
        uint32_t b = bytes - off < piece ? bytes - off : piece;
        bulk_g2s(static_cast<uint8_t *>(dst) + off, static_cast<const uint8_t *>(src) + off, b, bar);
    }
}

// ---- tensor memory (TMEM) as per-thread scratch: the per-node R/A/Q values
// of the walk live there instead of in shared memory ----
__device__ __forceinline__ void tm_alloc(uint32_t *dst, uint32_t cols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tm_dealloc(uint32_t taddr, uint32_t cols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}

__device__ __forceinline__ void tm_st1(uint32_t taddr, uint32_t v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}

__device__ __forceinline__ void tm_wait_st()
{
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// N consecutive columns of this warp's lane quarter; the wait takes the
// registers as operands so no use is scheduled before the data has arrived
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t (&v)[N])
{
    if constexpr (N == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                     : "=r"(v[0]), "=r"(v[1])
                     : "r"(taddr));
    } else {
        static_assert(N == 4, "2 or 4 columns");
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(taddr));
    }
}

template <int N>
__device__ __forceinline__ void tm_wait_ld(uint32_t (&a)[N], uint32_t (&b)[N])
{
    if constexpr (N == 2) {
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(a[0]), "+r"(a[1]), "+r"(b[0]), "+r"(b[1])::"memory");
    } else {
        asm volatile("tcgen05.wait::ld.sync.aligned;"
                     : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(b[0]), "+r"(b[1]),
                       "+r"(b[2]), "+r"(b[3])::"memory");
    }
}

// the low or high 16-bit half of a TMEM word, zero-extended: one PRMT
__device__ __forceinline__ int tm_half(uint32_t w, int hi) { return (int)__byte_perm(w, 0u, hi ? 0x4432u : 0x4410u); }

struct LbArgs {
    const uint8_t *tables; // groups x group_bytes
    const int32_t *ptm;    // [n][mp4] int32, ptm_bytes
    const uint16_t *prefix;
    const int32_t *depth;
    int32_t *lb_out;
    int *err;
    long long pool;
    const long long *pool_dev; // if set, the pool size is read on the device (B&B)
    fsp_lb_layout L;
    int groups, ppg;       // couple groups, couples per group
    int n, m, P, mp4, nrec;
    int stride;
    uint32_t hi_mul;       // 0x10000 (see mask_addr)
    const int32_t *cin;    // optional prefix completion times [pool][cin_stride]
    int cin_stride;
    int vec_rows;          // vectorised scheduled-set build (long prefixes)
    uint32_t tm_cols;      // TMEM columns allocated per CTA (TM variants)
    int dbuf;              // couple-group buffers (>= 2: multi-buffered, no CTA barrier)
    int woff;              // 16-bit walk offset D (= max p): e + D is carried
    int split;             // warps per tile (power of two <= W): each walks every
                           // split-th couple, LBs combined by atomicMax (lb_out zeroed)
    int tail_split;        // split of the last (partial) tile iteration (1: none);
                           // its nodes' lb_out entries are zeroed by the host
    unsigned long long *prof; // diagnostics (FSP_LB_PROF): per-phase SM cycles, summed
    uint32_t wait_ns;      // mbarrier try_wait suspend-time hint (0: none)
    const uint16_t *ulist; // B&B pools (nullable): node i's unscheduled jobs, n - depth[i]
                           // entries of row i (same stride); the prefix is then not read
                           // (completion times come from cin): rows start empty and each
                           // lane SETS its node's bits (deep nodes: n' << d entries)
    int lane_ingest;       // scheduled-set build with one node per lane (byte and
                           // lane-major rows); 0: the warp-per-node pass
    int sort_depth;        // fused dense path: the tile's nodes ranked by depth over the slots
    int jp;                // job-pair heads (fsp_lb_plan::jp): s_pq holds the job-pair rows
                           // and the C pass reads 16-bit PTM pair rows
    int prow;              // u32 words per PTM row in shared memory (fsp_ptm_row_words)
    int ptm8;              // jp plans: 8-bit PTM rows (step8)
    int jp_off;            // u32 words from PTM to the job-pair (or pq) rows
    uint32_t ltot2[16];    // per machine pair: sum_j p_j,2i | sum_j p_j,2i+1 << 16 (jp loads)
    uint32_t jp_m;         // their masking offset M (multiple of 16)
    uint32_t one;          // 1 (a multiplier ptxas keeps on the FMA pipe)
    int dbg_skip;          // diagnostics only (FSP_LB_DEBUG_SKIP): bit 0 skips the
                           // per-node heads phase, bit 1 the couple walks, bit 2 the
                           // job-pair heads (C pass only), bit 3 the C pass (LBs wrong)
};

// FSP_LB_PROF phases: cycles lane 0 of every warp spends in each part
enum { PR_INGEST = 0, PR_HEADS, PR_WAIT, PR_WALK, PR_RELEASE, PR_STORE, PR_N };

// Shared address of U[job][warp] from a record's meta word, whose address
// field is the row's byte offset; wst = the shared-window address of this
// warp's row segment (the kernel's own, nothing baked in by the host).
//   int32 form: meta = (c2 << 16) | off     -> (meta & 0xffff) + wst  (one IADD3)
//   s16 form:   meta = (off << 16) | c2     -> (meta >> 16) + wst     (one IMAD.HI)
// (hi_mul = 0x10000 arrives as a kernel argument so ptxas keeps an IMAD.HI on
// the FMA pipe instead of strength-reducing it to an ALU LEA.HI: the ALU pipe
// is the walk's bottleneck.)
template <bool S16>
__device__ __forceinline__ uint32_t mask_addr(uint32_t meta, uint32_t wst, uint32_t hi_mul,
                                              uint64_t wst64)
{
    // s16: one IMAD.WIDE.U32 with the loop-invariant 64-bit addend wst << 32
    // (a 32-bit "hi + c" form makes ptxas rebuild the {0, c} pair every time)
    if constexpr (S16) return (uint32_t)(((uint64_t)meta * hi_mul + wst64) >> 32);
    else return (meta & 0xffffu) + wst;
}

// U row layouts (one row per job, one segment per warp):
//  * lane-major (int32 walk): NPL words, bit L of word q = node q*32+L;
//  * byte (16-bit walk, m >= 10, BYTE): lane L owns byte L of the warp's
//    8-word row segment; bit 1+q of the byte = node q*32+L.  A lane loads its
//    byte (LDS.U8, zero-extended: no shift) and R2P turns bits 1..NPL into the
//    predicates P1..P4 of the updates (instead of one LOP3 per node);
//  * nibble (16-bit walk, m >= 10, !BYTE: long job lists, where 32 bytes per
//    row and warp do not fit): lane L owns NPL+1 bits of word L/LPW at shift
//    1 + (L % LPW)*(NPL+1); bit 1+q of the field = node q*32+L.  A lane loads
//    one word and shifts it by a multiply-high (FMA pipe) before the R2P.
template <int NPL, bool BYTE>
struct Nib {
    static constexpr int LPW = BYTE ? 4 : 31 / (NPL + 1);    // lanes per word
    static constexpr int WPR = (32 + LPW - 1) / LPW;          // words per warp segment
};

template <bool S16, int NPL, int MAXM, bool BYTE>
struct ULayout {
    // byte / nibble rows where the couple walk dominates (m >= 10); lane-major
    // rows for m = 5, where the per-node phase dominates (measured on 20x5)
    static constexpr bool NIB = S16 && MAXM >= 10;
    static constexpr bool BYTES = NIB && BYTE;
    static constexpr int WPR = NIB ? Nib<NPL, BYTE>::WPR : NPL;
    __device__ static int word(int L, int q) { return NIB ? L / Nib<NPL, BYTE>::LPW : q; }
    __device__ static int bit(int L, int q)
    {
        return !NIB ? L : BYTE ? (L % 4) * 8 + 1 + q : (L % Nib<NPL, BYTE>::LPW) * (NPL + 1) + 2 + q;
    }
};

// The NPL unscheduled-bit words of one job for this warp's NPL*32 nodes.
template <int NPL>
struct Mask {
    uint32_t b[NPL];
};

template <int NPL, bool BYTE = false>
__device__ __forceinline__ Mask<NPL> lds_mask(uint32_t addr)
{
    Mask<NPL> v;
    if constexpr (BYTE) {
        static_assert(NPL == 1, "one byte per lane");
        asm("ld.shared.u8 %0, [%1];" : "=r"(v.b[0]) : "r"(addr));
    } else if constexpr (NPL == 1) {
        asm("ld.shared.u32 %0, [%1];" : "=r"(v.b[0]) : "r"(addr));
    } else if constexpr (NPL == 2) {
        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.b[0]), "=r"(v.b[1]) : "r"(addr));
    } else {
        static_assert(NPL == 4, "NPL is 1, 2 or 4");
        asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
            : "=r"(v.b[0]), "=r"(v.b[1]), "=r"(v.b[2]), "=r"(v.b[3])
            : "r"(addr));
    }
    return v;
}

// One update of Fig. 3 lines 10-15 for one node in the difference form
// e = t2 - t1:  t1 += p_jk;  t2 = max(t2, t1 + lag_j) + p_jl
// is  e = max(e + x_j, y_j)  with x_j = p_jl - p_jk, y_j = lag_j + p_jl.  Line 10
// ("job not yet scheduled") is the predicate (a short branch ptxas predicates).
//   int32: e = max(e + x, y)  (x = top half of meta, extracted once per position)
//   16-bit: the low halfword carries e + D, D = max p (the walk offset):
//          0 <= e <= t2 <= (n+m-1)*max p and e + x >= 0 with x >= -max p, so
//          e + D and e + D + x stay in [0, 65535] (host-checked) and
//          e + D = max.u16(e + D + meta, c1) (VIADDMNMX.U16x2; the low halves
//          are x and y + D, the high halves only collect garbage that never
//          reaches the low one)
template <bool S16>
__device__ __forceinline__ void upd(uint32_t bits, uint32_t lanebit, uint32_t c1, uint32_t x,
                                    int &e)
{
    if (bits & lanebit) {
        asm volatile(""); // keep the branch so ptxas predicates the op
        if constexpr (S16) e = (int)__viaddmax_u16x2((unsigned)e, x, c1);
        else e = __viaddmax_s32(e, (int)x, (int)c1);
    }
}

// nibble layout: one word per lane (MW = 1); lane-major: NPL words
#define FSP_MASK(META) lds_mask<MW, UL::BYTES>(mask_addr<S16>((META), wst, hi_mul, wst64))
#define FSP_UPD(MASK, C1, META)                                                 \
    {                                                                           \
        const uint32_t x_ = S16 ? (META) : (uint32_t)((int)(META) >> 16);       \
        if constexpr (UL::NIB) {                                                \
            /* byte rows: the lane's byte; nibble rows: shifted by a mul-hi */  \
            const uint32_t nb_ = UL::BYTES ? (MASK).b[0] : __umulhi((MASK).b[0], shmul); \
            _Pragma("unroll") for (int q_ = 0; q_ < NPL; ++q_)                  \
                upd<S16>(nb_, 2u << q_, (C1), x_, ee[q_]);                      \
        } else {                                                                \
            _Pragma("unroll") for (int q_ = 0; q_ < NPL; ++q_)                  \
                upd<S16>((MASK).b[q_], lanebit, (C1), x_, ee[q_]);              \
        }                                                                       \
    }

// Rows a2/a3 of one node (lane's node q) over job PAIRS (2i, 2i+1), dense TMEM
// plans (fsp_lb_plan::jp).  Each 16x2 op carries both jobs of a pair for the
// node: job 2i in the low half, 2i+1 in the high half.  A scheduled job's half
// starts at M (a multiple of 16 above every real head and tail, host-checked
// with M + sum_k p_jk <= 65535), so it never wins a minimum and no branch or
// predicate is needed:
//   r_j0 = max(C_0, M2),  r_jk = max(C_k, r_j,k-1 + p_j,k-1)   (R3)   -> RR_k = min
//   t_j,m-1 = M2,  t_jl = t_j,l+1 + p_j,l+1  (= q_jl + M2, R4)       -> QQ_l = min
//   L_k = sum p_jk over unscheduled j: one multiply-add per machine with the
//   swapped flags (a_hi | a_lo << 16) x (p_lo | p_hi << 16), whose high half
//   is a_hi p_hi + a_lo p_lo (the low half collects <= ceil(n/2) max p, host-
//   checked against a carry)
// Per pair: 2 x m - 1 ALU ops for the heads, m - 1 for the tails, ~4 for the
// flags; the loads' and the tails' running sums are FMA-pipe multiply-adds.
// Returns true for a malformed node (unscheduled count != n - depth).
// Bitonic sort of the warp's 32*NPL keys, key q of lane L at position q*32+L
// (in-lane stages exchange registers, cross-lane stages shfl.xor), ascending.
template <int NPL>
__device__ __forceinline__ void warp_sort(uint32_t (&e)[NPL], int lane)
{
    constexpr int N = 32 * NPL;
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jq = j >> 5;
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    if ((q & jq) == 0) {
                        const int q2 = q | jq;
                        const bool asc = (((q * 32 + lane) & k) == 0);
                        const uint32_t lo = min(e[q], e[q2]), hi = max(e[q], e[q2]);
                        e[q] = asc ? lo : hi;
                        e[q2] = asc ? hi : lo;
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, e[q], j);
                    const bool asc = (((q * 32 + lane) & k) == 0);
                    const bool keep_min = ((lane & j) == 0) == asc;
                    e[q] = keep_min ? min(e[q], o) : max(e[q], o);
                }
            }
        }
    }
}

// TM: R/A/Q to tensor memory as machine pairs (column (arr*HM + k/2)*NPLP + q);
// else to the warp's shared arrays Rs/As/Qs [MAXM][TN] (16-bit), node q*32+lane.
// LC: the loads L_k come from the C pass (Lp = the prefix's machine-pair sums,
// L = total - Lp) instead of one multiply-add per machine and job here (the
// pools whose completion times are supplied, cin, have no C pass).
template <int MAXM, int HM, int NPLP, class UL, bool TM, int TN, bool LC>
__device__ __forceinline__ bool jp_heads(const LbArgs &a, const uint32_t *s_jp, const uint32_t *Uw,
                                         int urow, int useg, int lane, int q, const int (&C)[MAXM],
                                         const uint32_t (&Lp)[HM], uint32_t tbase, uint16_t *Rs, int n,
                                         int want)
{
    constexpr int MP4 = (MAXM + 3) & ~3;
    uint32_t C2[MAXM], RR[MAXM], QQ[MAXM], LL[MAXM];
#pragma unroll
    for (int k = 0; k < MAXM; ++k) {
        C2[k] = (uint32_t)C[k] * 0x10001u;
        RR[k] = QQ[k] = 0xffffffffu;
        LL[k] = 0u;
    }
    const uint32_t M = a.jp_m, MM = M * 0x10001u, one = a.one;
    const int sh = UL::bit(lane, q);
    const uint32_t *uw = Uw + useg + UL::word(lane, q);
    uint32_t cnt2 = 0;
    const int npair = (n + 1) >> 1; // row n of U is the always-empty padding row
    int i = 0;
#if FSP_JP2
    // two pairs per iteration: their heads and tails fold into the minima with
    // one 3-input VIMNMX3.U16x2 per machine (the forward pass does the heads
    // and the loads, the backward pass reloads the rows for the tails)
    auto flags = [&](int ip, uint32_t &ab, uint32_t &absw, uint32_t &M2) {
        if constexpr (UL::BYTES && FSP_JP_BYTEFLAGS) {
            // byte rows: the lane's two bytes, merged into one word by a PRMT, one
            // shift and one mask give both flags at bits 0 and 16
            const uint8_t *ub = reinterpret_cast<const uint8_t *>(Uw + useg) + lane;
            const uint32_t w = __byte_perm((uint32_t)ub[(2 * ip) * urow * 4], (uint32_t)ub[(2 * ip + 1) * urow * 4],
                                           0x1410u);
            ab = (w >> (1 + q)) & 0x10001u;
            absw = __byte_perm(ab, ab, 0x1032u);
        } else {
            const uint32_t xl = uw[(2 * ip) * urow], xh = uw[(2 * ip + 1) * urow];
            const uint32_t bl = (xl >> sh) & 1u, bh = (xh >> sh) & 1u;
            ab = bl | (bh << 16);
            absw = bh | (bl << 16);
        }
        M2 = MM - ab * M;
    };
    auto ldrow = [&](int ip, int k4) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"((uint32_t)__cvta_generic_to_shared(s_jp + (size_t)ip * MP4 + 4 * k4)));
        return v;
    };
#pragma unroll 1
    for (; MAXM >= 10 && i + 1 < npair; i += 2) { // (5 machines: one pair at a time, measured)
        uint32_t abA, abswA, M2A, abB, abswB, M2B;
        flags(i, abA, abswA, M2A);
        flags(i + 1, abB, abswB, M2B);
        cnt2 += abA + abB;
        uint32_t rA = __vmaxu2(C2[0], M2A), rB = __vmaxu2(C2[0], M2B);
        RR[0] = __vimin3_u16x2(RR[0], rA, rB);
#pragma unroll
        for (int k4 = 0; k4 < MP4 / 4; ++k4) {
            const uint4 va = ldrow(i, k4), vb = ldrow(i + 1, k4);
            const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int k = 4 * k4 + t;
                if (k < MAXM) {
                    if constexpr (!LC) {
                        LL[k] = wa[t] * abswA + LL[k];
                        LL[k] = wb[t] * abswB + LL[k];
                    }
                    if (k + 1 < MAXM) {
                        rA = __viaddmax_u16x2(rA, wa[t], C2[k + 1]);
                        rB = __viaddmax_u16x2(rB, wb[t], C2[k + 1]);
                        RR[k + 1] = __vimin3_u16x2(RR[k + 1], rA, rB);
                    }
                }
            }
        }
#if !FSP_JP_SPLIT
        uint32_t tA = M2A, tB = M2B;
#pragma unroll
        for (int k4 = MP4 / 4 - 1; k4 >= 0; --k4) {
            const uint4 va = ldrow(i, k4), vb = ldrow(i + 1, k4);
            const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
            for (int t = 3; t >= 0; --t) {
                const int k = 4 * k4 + t; // QQ[k-1] = min over jobs of q_j,k-1 + M2 = t after + p_jk
                if (k >= 1 && k < MAXM) {
                    tA = wa[t] * one + tA;
                    tB = wb[t] * one + tB;
                    QQ[k - 1] = __vimin3_u16x2(QQ[k - 1], tA, tB);
                }
            }
        }
#endif
    }
#if FSP_JP_SPLIT
    // tails in a second pass over the pairs (fewer live registers per pass:
    // no spills in either loop)
#pragma unroll 1
    for (int i2 = 0; MAXM >= 10 && i2 + 1 < npair; i2 += 2) {
        uint32_t abA, abswA, M2A, abB, abswB, M2B;
        flags(i2, abA, abswA, M2A);
        flags(i2 + 1, abB, abswB, M2B);
        uint32_t tA = M2A, tB = M2B;
#pragma unroll
        for (int k4 = MP4 / 4 - 1; k4 >= 0; --k4) {
            const uint4 va = ldrow(i2, k4), vb = ldrow(i2 + 1, k4);
            const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
            for (int t = 3; t >= 0; --t) {
                const int k = 4 * k4 + t;
                if (k >= 1 && k < MAXM) {
                    tA = wa[t] * one + tA;
                    tB = wb[t] * one + tB;
                    QQ[k - 1] = __vimin3_u16x2(QQ[k - 1], tA, tB);
                }
            }
        }
    }
#endif
#endif
#pragma unroll 1
    for (; i < npair; ++i) {
        const uint32_t xl = uw[(2 * i) * urow], xh = uw[(2 * i + 1) * urow];
        const uint32_t bl = (xl >> sh) & 1u, bh = (xh >> sh) & 1u;
        const uint32_t ab = bl | (bh << 16), absw = bh | (bl << 16);
        const uint32_t M2 = MM - ab * M;
        cnt2 += ab;
        const uint4 *pr = reinterpret_cast<const uint4 *>(s_jp + (size_t)i * MP4);
        uint32_t pw[MP4];
#pragma unroll
        for (int k4 = 0; k4 < MP4 / 4; ++k4) {
            const uint4 v = pr[k4];
            pw[4 * k4] = v.x;
            pw[4 * k4 + 1] = v.y;
            pw[4 * k4 + 2] = v.z;
            pw[4 * k4 + 3] = v.w;
        }
        uint32_t r = __vmaxu2(C2[0], M2);
        RR[0] = __vminu2(RR[0], r);
#pragma unroll
        for (int k = 1; k < MAXM; ++k) {
            r = __viaddmax_u16x2(r, pw[k - 1], C2[k]);
            RR[k] = __vminu2(RR[k], r);
        }
        uint32_t t = M2;
#pragma unroll
        for (int l = MAXM - 2; l >= 0; --l) {
            QQ[l] = __viaddmin_u16x2(t, pw[l + 1], QQ[l]);
            t = pw[l + 1] * one + t;
        }
        if constexpr (!LC) {
#pragma unroll
            for (int k = 0; k < MAXM; ++k) LL[k] = pw[k] * absw + LL[k];
        }
    }
    const int cnt = (int)((cnt2 & 0xffffu) + (cnt2 >> 16));
    if constexpr (LC) { // L_k in the high halves, as the multiply-adds leave them
#pragma unroll
        for (int k = 0; k < MAXM; ++k) {
            const uint32_t l2 = a.ltot2[k >> 1] - Lp[k >> 1]; // no borrow: every half total >= prefix
            LL[k] = (k & 1) ? (l2 & 0xffff0000u) : (l2 << 16);
        }
    }
    if constexpr (!TM) {
        uint16_t *As = Rs + MAXM * TN, *Qs = As + MAXM * TN;
#pragma unroll
        for (int k = 0; k < MAXM; ++k) {
            const uint32_t r = __vminu2(RR[k], __byte_perm(RR[k], 0u, 0x1032));
            const uint32_t qv = k == MAXM - 1 ? 0u : __vminu2(QQ[k], __byte_perm(QQ[k], 0u, 0x1032));
            const uint32_t R = cnt ? (r & 0xffffu) : (C2[k] & 0xffffu); // R6: R = A = C, Q = 0
            Rs[k * TN + q * 32 + lane] = (uint16_t)R;
            As[k * TN + q * 32 + lane] = (uint16_t)(cnt ? R + (LL[k] >> 16) : R);
            Qs[k * TN + q * 32 + lane] = (uint16_t)(cnt ? qv & 0xffffu : 0u);
        }
        return cnt != want;
    } else {
        uint32_t R2[HM], A2[HM], Q2[HM];
#pragma unroll
        for (int kp = 0; kp < HM; ++kp) {
            const uint32_t r0 = RR[2 * kp], r1 = RR[2 * kp + 1];
            const uint32_t q0 = QQ[2 * kp], q1 = 2 * kp + 1 == MAXM - 1 ? 0u : QQ[2 * kp + 1];
            R2[kp] = __vminu2(__byte_perm(r0, r1, 0x5410), __byte_perm(r0, r1, 0x7632));
            Q2[kp] = __vminu2(__byte_perm(q0, q1, 0x5410), __byte_perm(q0, q1, 0x7632));
            A2[kp] = R2[kp] + __byte_perm(LL[2 * kp], LL[2 * kp + 1], 0x7632); // A = R + L
            if (cnt == 0) { // R6: complete schedule, R = C, A = C, Q = 0
                R2[kp] = A2[kp] = __byte_perm(C2[2 * kp], C2[2 * kp + 1], 0x5410);
                Q2[kp] = 0u;
            }
        }
#pragma unroll
        for (int kp = 0; kp < HM; ++kp) {
            tm_st1(tbase + (0 * HM + kp) * NPLP + q, R2[kp]);
            tm_st1(tbase + (1 * HM + kp) * NPLP + q, A2[kp]);
            tm_st1(tbase + (2 * HM + kp) * NPLP + q, Q2[kp]);
        }
        return cnt != want;
    }
}

// launch bounds: 8 warps for m > 20; 4 warps x 5 CTAs per SM for m = 5 (the
// per-node phase dominates there: small CTAs, registers capped at 96 so five
// fit; measured 20x5: 5.0 G bounds/s vs 3.9 G with one 16-warp CTA); else 16
// RG (placement ablation, NEXT-3): the couple records are read from global
// memory (L1/L2, read-only path) instead of the TMA-staged shared buffers.
// KC (dense TMEM walks, short job lists: fsp_lb_plan::kcache): R_k and A_k are
// kept in registers while k is unchanged, as in the sparse walk (20x20 +5 %;
// at 200x20 the extra live registers cost 0.7 %, profiles/r02/dense_kcache_ab.txt)
template <int MAXM, bool EXACT, bool S16, int NPL, bool SPARSE, bool BYTE = true, bool RG = false, bool KC = false>
__global__ void __launch_bounds__(MAXM > 20 ? 256 : MAXM <= 5 ? 128 : 512, MAXM <= 5 ? 5 : 1)
    lb_kernel(const LbArgs a)
{
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int kUnroll = SPARSE ? FSP_WALK_UNROLL_SPARSE : MAXM <= 5 ? 1 : KC ? 4 : FSP_WALK_UNROLL_DENSE;
    if (a.pool_dev && *a.pool_dev == 0) return; // B&B: an empty (or rerouted) pool
    const int n = a.n;
    const int m = EXACT ? MAXM : a.m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    constexpr int TN = 32 * NPL;                                         // nodes per warp
    // U: lane-major rows [(n+1)][W][NPL] (records hold absolute addresses), or,
    // nibble layout, one block per warp [W][(n+1)][urow] (records hold the row
    // offset, the warp's block base is added per visit: no 64 KB limit on W)
    uint32_t *Uw = reinterpret_cast<uint32_t *>(smem + a.L.off_u) +
                   (ULayout<S16, NPL, MAXM, BYTE>::NIB ? (size_t)warp * (n + 1) * a.L.urow_words : 0);
    const int32_t *s_ptm = reinterpret_cast<const int32_t *>(smem + a.L.off_ptm);
    // TM variants: per job [p pairs x HMP][q pairs x HMP] u32 after PTM (see fsp_plan_lb)
    // jp plans: PTM rows of packed 16-bit machine pairs (a.prow words), then the
    // job-pair rows; else int32 rows (mp4 words), then the (p, q) pair rows
    const uint32_t *s_pq = reinterpret_cast<const uint32_t *>(s_ptm + (size_t)a.jp_off);
    uint64_t *s_bar = reinterpret_cast<uint64_t *>(smem + a.L.off_bar);
    // per-warp heads R[MAXM][TN], A = R + L [MAXM][TN] (L_k = sum of p_jk over
    // the unscheduled jobs) and tails Q[MAXM][TN]; int16 in the s16 walk (all
    // values fit, host-checked), int32 otherwise
    using rt_t = typename std::conditional<S16, uint16_t, int32_t>::type;
    rt_t *Rs = reinterpret_cast<rt_t *>(smem + a.L.off_rt + (size_t)warp * a.L.rt_bytes);
    rt_t *As = Rs + MAXM * TN;
    rt_t *Qs = As + MAXM * TN;
    uint8_t *s_tab = smem + a.L.off_tab;
    // SPARSE: per-warp list of the couple's records whose job is unscheduled in
    // at least one of the warp's nodes (the walk over the others is a no-op)
    uint2 *s_list = reinterpret_cast<uint2 *>(smem + a.L.off_list + (size_t)warp * a.L.list_bytes);

    // TM: the per-node R, A, Q of phase A go to tensor memory, two machines per
    // 32-bit column (16-bit values): column (arr*HM + k/2)*NPL + q of this
    // warp's block in its lane quarter (warp % 4), blocks of TCOLS columns
    constexpr bool TM = ULayout<S16, NPL, MAXM, BYTE>::NIB;
    constexpr int NPLP = NPL; // TMEM columns per (array, machine pair)
    constexpr int HM = (MAXM + 1) / 2, TCOLS = 3 * HM * NPLP;
    constexpr int HMP = (HM + 3) & ~3; // machine pairs per packed row, padded to 16 bytes
    // barrier area (32 B per buffer): mbarriers "group buffer b full" (b = 0 also
    // counts PTM), mbarriers "buffer b released by all warps", release counters,
    // TMEM base address
    uint64_t *s_emp = s_bar + FSP_MAX_GBUF;
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(s_emp + FSP_MAX_GBUF);
    uint32_t *s_tm = s_cnt + FSP_MAX_GBUF;
    if constexpr (TM) {
        if (warp == 0) tm_alloc(s_tm, a.tm_cols);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }

    auto group_size = [&](int g) {
        int np = a.P - g * a.ppg;
        return np < a.ppg ? np : a.ppg;
    };
    auto group_blob = [&](int g) {
        if (a.L.pos_off) return (uint32_t)a.L.group_bytes; // + the inverse position table
        return (uint32_t)((a.L.kl_bytes +
                           ((size_t)group_size(g) * a.nrec + FSP_REC_SLACK) * sizeof(fsp_rec) + 15) &
                          ~size_t(15));
    };

    const long long pool = a.pool_dev ? *a.pool_dev : a.pool;
    const long long ntiles = (pool + TN - 1) / TN;
    // small pools (fewer tiles than warps on the GPU): `split` warps share a
    // tile, each walking every split-th couple of a group (phase A is repeated
    // per warp); warps split*t .. split*t+split-1 sit on different SMSPs
    const int Wt = W / a.split; // tiles per CTA iteration
    const long long niter = (ntiles + (long long)Wt * gridDim.x - 1) / ((long long)Wt * gridDim.x);
    // double-buffered couple groups: the CTA's sequence of groups is it*G + gi;
    // group sequence number sq lives in buffer sq % NB, whose (sq / NB)-th fill
    // it is; the last warp to release a buffer refills it with group sq + NB
    // (a warp runs at most NB - 1 groups ahead of the slowest of its CTA)
    const int NB = a.dbuf;
    const bool dbuf = NB >= 2;
    const int woff = S16 ? a.woff : 0;
    const long long nseq = niter * a.groups;

    // ---- stage PTM + the first couple group(s) (TMA bulk, mbarriers) ----
    if (threadIdx.x == 0) {
        for (int b = 0; b < FSP_MAX_GBUF; ++b) {
            mbar_init(s_bar + b, 1);
            mbar_init(s_emp + b, W);
            s_cnt[b] = 0;
        }
        uint32_t gb = RG ? 0u : group_blob(0);
        mbar_expect_tx(s_bar, gb + (uint32_t)a.L.ptm_bytes);
        if (!RG) bulk_copy(s_tab, a.tables, gb, s_bar);
        bulk_copy(smem + a.L.off_ptm, a.ptm, (uint32_t)a.L.ptm_bytes, s_bar);
        for (int b = 1; !RG && dbuf && b < NB && b < nseq; ++b) {
            const int g = b % a.groups;
            gb = group_blob(g);
            mbar_expect_tx(s_bar + b, gb);
            bulk_copy(s_tab + (size_t)b * a.L.group_bytes, a.tables + (size_t)g * a.L.group_bytes, gb,
                      s_bar + b);
        }
    }
    __syncthreads();
    uint32_t tbase = 0;
    if constexpr (TM) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tbase = *s_tm + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * TCOLS);
    }
    uint32_t phase = 0;
    mbar_wait(s_bar, phase);
    phase ^= 1;
    int resident = 0;

    // iteration `it` of CTA b takes tiles (it*Wt + warp/split)*grid + b: the
    // tiles of a partial last iteration spread over every SM (a few idle warps
    // per CTA) instead of leaving whole SMs idle
    const uint32_t lanebit = 1u << lane;
    using UL = ULayout<S16, NPL, MAXM, BYTE>;
    constexpr int WPR = UL::WPR;                 // U words per warp per job row
    constexpr int MW = UL::NIB ? 1 : NPL;        // mask words a lane loads
    const int lw = UL::word(lane, 0);            // nibble layout: this lane's word
    // byte rows: the lane's mask byte is at byte offset `lane` of the row
    // segment; nibble rows: the lane's word, shifted (lsh >= 1) to bits 1..NPL by
    // a multiply-high by 2^(32 - lsh) on the FMA pipe
    const int lsh = (UL::NIB && !UL::BYTES) ? UL::bit(lane, 0) - 1 : 1;
    const uint32_t shmul = 1u << (32 - lsh);
    const uint32_t wst = UL::BYTES ? smem_u32(Uw) + (uint32_t)lane
                         : UL::NIB ? smem_u32(Uw) + 4u * lw : smem_u32(Uw) + 4u * (WPR * warp);
    const int urow = a.L.urow_words; // words per job row of U (padded against bank conflicts)
    const uint32_t hi_mul = a.hi_mul;
    const uint64_t wst64 = (uint64_t)wst << 32;
    const int useg = UL::NIB ? 0 : WPR * warp; // this warp's segment of a U row

    long long pt = a.prof ? clock64() : 0;
    auto mark = [&](int ph) {
        if (a.prof) {
            const long long t = clock64();
            if (lane == 0) atomicAdd(&a.prof[ph], (unsigned long long)(t - pt));
            pt = t;
        }
    };
    for (long long it = 0; it < niter; ++it) {
        // the last, partial iteration may split its tiles over more warps (a
        // partial wave otherwise leaves most warps of every SM idle)
        const int split = it + 1 == niter && a.tail_split > a.split ? a.tail_split : a.split;
        const int slice = warp & (split - 1);
        const long long tile = it * Wt * gridDim.x + (long long)(warp / split) * gridDim.x + blockIdx.x;
        bool bad = false;

        // ---------------- a1: node ingest (depth, scheduled set) ----------------
        // slot (q, lane) holds node tile*TN + sidx[q]: q*32 + lane, or, with the
        // fused C pass (a.sort_depth), the tile's nodes ranked by depth, so the
        // 32 prefixes a C-pass step walks together are about equally long (the
        // pass runs to the deepest of them)
        const bool fused = !SPARSE && !a.cin && a.lane_ingest && (!UL::NIB || UL::BYTES);
        int dq[NPL];
        uint32_t sidx[NPL];
        uint32_t validq[NPL];
        uint32_t anyvalid = 0;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const long long node = tile * TN + q * 32 + lane;
            const bool has = node < pool;
            int d = has ? FSP_LDS_STREAM(a.depth + node) : 0; // streamed: read once (evict-first)
            if (d < 0 || d > n || d > a.stride) {
                bad = true;
                d = 0;
            }
            dq[q] = d;
            sidx[q] = (uint32_t)(q * 32 + lane);
        }
        if (fused && a.sort_depth) {
            uint32_t key[NPL];
#pragma unroll
            for (int q = 0; q < NPL; ++q) key[q] = ((uint32_t)dq[q] << 8) | sidx[q];
            warp_sort<NPL>(key, lane);
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                dq[q] = (int)(key[q] >> 8);
                sidx[q] = key[q] & 0xffu;
            }
        }
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            validq[q] = __ballot_sync(0xffffffffu, tile * TN + sidx[q] < pool);
            anyvalid |= validq[q];
        }
        // all-unscheduled pattern of this warp's segment
        uint32_t pat[WPR];
        if constexpr (UL::NIB) {
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < NPL; ++q)
                if ((validq[q] >> lane) & 1u) mine |= 1u << UL::bit(lane, q);
#pragma unroll
            for (int w = 0; w < WPR; ++w) pat[w] = __reduce_or_sync(0xffffffffu, lw == w ? mine : 0u);
        } else {
#pragma unroll
            for (int q = 0; q < NPL; ++q) pat[q] = validq[q];
        }
        for (int j = lane; j <= n; j += 32) {
#pragma unroll
            for (int w = 0; w < WPR; ++w) // row n: the padding record's always-empty mask
                Uw[j * urow + useg + w] = j < n && !a.ulist ? pat[w] : 0u;
        }
        __syncwarp();
        // dense pools whose prefix completion times are computed here (no cin):
        // each lane clears its node's bits in the same pass over the prefix
        // that computes C (phase A below), reading every prefix once (fused)
        if (fused) {
            // (scheduled bits cleared in phase A)
        } else if (a.lane_ingest && !UL::NIB || a.lane_ingest && UL::BYTES) {
            // each lane clears the bits of its own nodes: byte rows give lane L
            // byte L of the row segment (plain byte stores, no other lane
            // touches it); lane-major rows share a word per 32 nodes (shared
            // atomics).  All lanes' row loads are in flight at once (one row
            // per lane, 16-byte vectors) instead of one node at a time.
            uint8_t *ub = reinterpret_cast<uint8_t *>(Uw + useg) + lane;
            const int urowB = urow * 4;
            const bool setm = UL::BYTES && a.ulist != nullptr; // set unscheduled bits instead
            const uint16_t *src = setm ? a.ulist : a.prefix;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const long long node = tile * TN + q * 32 + lane;
                const int d = setm ? (node < pool ? n - dq[q] : 0) : dq[q];
                const uint16_t *row = src + (size_t)node * a.stride;
                const bool v16 = ((reinterpret_cast<uintptr_t>(src) | ((uintptr_t)a.stride * 2)) & 15) == 0;
                auto clear = [&](uint32_t job) {
                    if (job < (uint32_t)n) {
                        if constexpr (UL::BYTES) {
                            if (setm) ub[job * urowB] |= (uint8_t)(2u << q);
                            else ub[job * urowB] &= (uint8_t)~(2u << q);
                        } else {
                            atomicAnd(&Uw[job * urow + useg + q], ~lanebit);
                        }
                    }
                };
                int i = 0;
                if (v16) {
                    const uint4 *r4 = reinterpret_cast<const uint4 *>(row);
                    for (; i + 16 <= d; i += 16) { // two vectors in flight
                        const uint4 v0 = FSP_LDS_STREAM(r4 + (i >> 3)), v1 = FSP_LDS_STREAM(r4 + (i >> 3) + 1);
                        const uint32_t w8[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            clear(w8[t] & 0xffffu);
                            clear(w8[t] >> 16);
                        }
                    }
                    if (i < d) {
                        const uint4 v0 = r4[i >> 3];
                        const uint4 v1 = i + 8 < d ? r4[(i >> 3) + 1] : v0;
                        const uint32_t w8[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                        for (int t = 0; t < 16; ++t)
                            if (i + t < d) clear(t & 1 ? w8[t >> 1] >> 16 : w8[t >> 1] & 0xffffu);
                    }
                } else {
                    for (; i < d; ++i) clear(row[i]);
                }
            }
            __syncwarp();
        } else {
        // coalesced pass over the TN prefix records: clear the scheduled bits
            // (16-byte rows: each lane takes eight job ids per vector load; the
            // next node's row is loaded while this one's bits are cleared)
            const bool rows16 = a.vec_rows && ((reinterpret_cast<uintptr_t>(a.prefix) | ((uintptr_t)a.stride * 2)) & 15) == 0;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                if (rows16) {
                    // segment `sg` of node L's row: entries 256*sg .. 256*sg+255
                    auto load_row = [&](int L, int sg) {
                        const int dL = __shfl_sync(0xffffffffu, dq[q], L);
                        uint4 v = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                        if (sg * 256 + lane * 8 < dL)
                            v = reinterpret_cast<const uint4 *>(a.prefix + (size_t)(tile * TN + q * 32 + L) *
                                                                               a.stride)[sg * 32 + lane];
                        return v;
                    };
                    // the first segment of the next node is loaded while this
                    // node's bits are cleared
                    uint4 cur = load_row(0, 0);
                    for (int L = 0; L < 32; ++L) {
                        const int dL = __shfl_sync(0xffffffffu, dq[q], L);
                        const uint32_t clr = ~(1u << UL::bit(L, q));
                        const int uwd = useg + UL::word(L, q);
                        const uint4 nxt = L + 1 < 32 ? load_row(L + 1, 0) : cur;
                        for (int sg = 0; sg * 256 < dL; ++sg) {
                            if (sg > 0) cur = load_row(L, sg);
                            const uint32_t w4[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                const uint32_t job = (t & 1) ? (w4[t >> 1] >> 16) : (w4[t >> 1] & 0xffffu);
                                if (sg * 256 + lane * 8 + t < dL && job < (uint32_t)n)
                                    Uw[job * urow + uwd] &= clr;
                            }
                        }
                        __syncwarp();
                        cur = nxt;
                    }
                } else {
                    for (int L = 0; L < 32; ++L) {
                        const int dL = __shfl_sync(0xffffffffu, dq[q], L);
                        if (dL == 0) continue;
                        const uint16_t *row = a.prefix + (size_t)(tile * TN + q * 32 + L) * a.stride;
                        const uint32_t clr = ~(1u << UL::bit(L, q));
                        const int uwd = useg + UL::word(L, q);
                        for (int i = lane; i < dL; i += 32) {
                            const uint32_t job = row[i];
                            if (job < (uint32_t)n) Uw[job * urow + uwd] &= clr;
                        }
                        __syncwarp();
                    }
                }
            }
        }

        // live jobs: unscheduled in at least one node of this warp; lane w keeps
        // the bitset word of jobs 32w .. 32w+31 (n <= 1024 for the sparse plan)
        int live = n;
        uint32_t livew = 0;
        if constexpr (SPARSE) {
            live = 0;
            for (int j0 = 0; j0 < n; j0 += 32) {
                const int j = j0 + lane;
                uint32_t any = 0;
                if (j < n) {
#pragma unroll
                    for (int w = 0; w < WPR; ++w) any |= Uw[j * urow + useg + w];
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, any != 0);
                if (lane == (j0 >> 5)) livew = bal;
                live += __popc(bal);
            }
        }
        const bool compact = SPARSE && live + 16 <= n;
        // few live jobs (deep B&B blocks): compaction by the inverse position
        // table (plan with pos_off), lane t < live holding the t-th live job
        const bool inv = SPARSE && compact && live <= 32 && a.L.pos_off != 0;
        int jt = 0;
        if constexpr (SPARSE) {
            if (inv) {
                int base = 0;
                for (int w0 = 0; w0 * 32 < n; ++w0) {
                    const uint32_t bits = __shfl_sync(0xffffffffu, livew, w0);
                    const int c = __popc(bits);
                    if (lane >= base && lane < base + c) jt = w0 * 32 + (int)__fns(bits, 0, lane - base + 1);
                    base += c;
                }
            }
        }

        mark(PR_INGEST);
        // ---------------- per node of this lane: C, heads, tails ----------------
#pragma unroll 1
        for (int q = 0; q < ((a.dbg_skip & 1) ? 0 : NPL); ++q) {
            int d = dq[0]; // (select chain: no local-memory indexing)
            uint32_t si = sidx[0];
#pragma unroll
            for (int t = 1; t < NPL; ++t)
                if (q == t) {
                    d = dq[t];
                    si = sidx[t];
                }
            const long long node = tile * TN + si;
            // prefix completion times C_k
            int C[MAXM];
#pragma unroll
            for (int k = 0; k < MAXM; ++k) C[k] = 0;
            const uint16_t *row = a.prefix + (size_t)(d ? node : 0) * a.stride;
            if (a.cin) { // completion times supplied (B&B children: parent C + one job)
                if (node < pool) {
                    const int32_t *cr = a.cin + (size_t)node * a.cin_stride;
                    if ((reinterpret_cast<uintptr_t>(cr) & 15) == 0) { // 16-byte rows: vectors
#pragma unroll
                        for (int k4 = 0; k4 < (MAXM + 3) / 4; ++k4) {
                            if (4 * k4 < m) {
                                const int4 v = reinterpret_cast<const int4 *>(cr)[k4];
                                const int cv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                                for (int t = 0; t < 4; ++t)
                                    if (4 * k4 + t < MAXM && 4 * k4 + t < m) C[4 * k4 + t] = cv[t];
                            }
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < MAXM; ++k)
                            if (k < m) C[k] = cr[k];
                    }
                }
            }
            const uint32_t one = a.one;
            // one job of the prefix: C_k = max(C_k, C'_k-1) + p_jk;
            // max(C_k, C'_k-1) + p = max(C'_k-1 + p, C_k + p): the second sum on
            // the FMA pipe (one * p + C), one VIADDMNMX on the ALU pipe
            auto step = [&](uint32_t job) {
                if (job >= (uint32_t)n) {
                    bad = true;
                    job = 0;
                }
                const int4 *pr = reinterpret_cast<const int4 *>(s_ptm + job * a.mp4);
                int prev = 0;
#pragma unroll
                for (int k4 = 0; k4 < (MAXM + 3) / 4; ++k4) {
                    if (4 * k4 < m) {
                        const int4 v = pr[k4];
                        const int pv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int k = 4 * k4 + t;
                            if (k < MAXM && k < m) {
                                C[k] = __viaddmax_s32(prev, pv[t], pv[t] * (int)one + C[k]);
                                prev = C[k];
                            }
                        }
                    }
                }
            };
            // jp plans: 16-bit PTM rows (half the gathered bytes), word i =
            // p_2i | p_2i+1 << 16; the chain runs in low halves (VIADDMNMX.U16x2,
            // the high halves collect garbage, masked off after the pass), odd
            // machines through a half swap
            // jp plans: machine-pair sums of the prefix's p (the loads L = total - Lp)
            uint32_t Lp[HM];
#pragma unroll
            for (int kp = 0; kp < HM; ++kp) Lp[kp] = 0u;
            auto step16 = [&](uint32_t job) {
                if (job >= (uint32_t)n) {
                    bad = true;
                    job = 0;
                }
                const uint4 *pr = reinterpret_cast<const uint4 *>(s_ptm + job * a.prow);
                uint32_t prev = 0;
#pragma unroll
                for (int c4 = 0; c4 < (MAXM / 2 + 3) / 4; ++c4) {
                    const uint4 v = pr[c4];
                    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int k = 2 * (4 * c4 + t);
                        if (k < MAXM) {
                            const uint32_t w = w4[t], ws = __byte_perm(w, w, 0x1032);
                            prev = __viaddmax_u16x2(prev, w, w * one + (uint32_t)C[k]);
                            C[k] = (int)prev;
                            Lp[k >> 1] = w * one + Lp[k >> 1];
                            if (k + 1 < MAXM) { // (odd m: the last machine has no pair)
                                prev = __viaddmax_u16x2(prev, ws, ws * one + (uint32_t)C[k + 1]);
                                C[k + 1] = (int)prev;
                            }
                        }
                    }
                }
            };
            const int dd = a.cin || (a.dbg_skip & 8) ? 0 : d;
            // fused ingest: also clear this node's bit of each scheduled job's
            // row (byte rows: lane-owned byte; lane-major: shared atomic)
            uint8_t *ubq = reinterpret_cast<uint8_t *>(Uw + useg) + lane;
            auto clr = [&](uint32_t job) {
                if (fused && job < (uint32_t)n) {
                    if constexpr (UL::BYTES) ubq[job * (urow * 4)] &= (uint8_t)~(2u << q);
                    else atomicAnd(&Uw[job * urow + useg + q], ~lanebit);
                }
            };
            // 8-bit rows (every p <= 255): one LDS.64 per 8 machines; each byte
            // pair becomes the (p_k | p_k+1 << 16) word and its swap by PRMT
            auto step8 = [&](uint32_t job) {
                if (job >= (uint32_t)n) {
                    bad = true;
                    job = 0;
                }
                const uint2 *pr = reinterpret_cast<const uint2 *>(s_ptm + job * a.prow);
                uint32_t prev = 0;
#pragma unroll
                for (int c8 = 0; c8 < (MAXM + 7) / 8; ++c8) {
                    const uint2 v = pr[c8];
                    const uint32_t w4[2] = {v.x, v.y};
#pragma unroll
                    for (int h = 0; h < 4; ++h) { // byte pairs (0,1) (2,3) of each word
                        const int k = 8 * c8 + 2 * h;
                        if (k < MAXM) {
                            const uint32_t src = w4[h >> 1];
                            const uint32_t w = __byte_perm(src, 0u, (h & 1) ? 0x4342u : 0x4140u);
                            const uint32_t ws = __byte_perm(src, 0u, (h & 1) ? 0x4243u : 0x4041u);
                            prev = __viaddmax_u16x2(prev, w, w * one + (uint32_t)C[k]);
                            C[k] = (int)prev;
                            Lp[k >> 1] = w * one + Lp[k >> 1];
                            if (k + 1 < MAXM) {
                                prev = __viaddmax_u16x2(prev, ws, ws * one + (uint32_t)C[k + 1]);
                                C[k + 1] = (int)prev;
                            }
                        }
                    }
                }
            };
            // the prefix pass with step function ST (no branch between the jobs
            // of a vector: the scheduler overlaps consecutive jobs' chains)
            auto pass = [&](auto &&st) {
                int i = 0;
                // 16-byte rows: eight job ids per vector load; the eight clears
                // follow the eight steps
                if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
                    const uint4 *r4 = reinterpret_cast<const uint4 *>(row);
                    for (; i + 8 <= dd; i += 8) {
                        // streamed (evict-first): each prefix is read once, the couple
                        // records the TMA ring re-reads stay in L2
                        const uint4 v = FSP_LDS_STREAM(r4 + (i >> 3));
                        const uint32_t w8[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int t = 0; t < 8; ++t) st(t & 1 ? w8[t >> 1] >> 16 : w8[t >> 1] & 0xffffu);
#pragma unroll
                        for (int t = 0; t < 8; ++t) clr(t & 1 ? w8[t >> 1] >> 16 : w8[t >> 1] & 0xffffu);
                    }
                }
                for (; i < dd; ++i) {
                    const uint32_t job = row[i];
                    clr(job);
                    st(job);
                }
            };
            int jform = 0; // 0: int32 rows, 1: 16-bit rows, 2: 8-bit rows (5 machines only:
                           // slower at 20 machines, profiles/r02/ptm8_ab.txt)
            if constexpr (!SPARSE && EXACT && S16) jform = a.jp ? (a.ptm8 && MAXM <= 5 ? 2 : 1) : 0;
            if constexpr (MAXM <= 5) {
                if (jform == 2) pass(step8);
                else if (jform == 1) pass(step16);
                else pass(step);
            } else {
                if (jform == 1) pass(step16);
                else pass(step);
            }
            if (fused) __syncwarp(); // every lane's bits of node group q cleared
            // a2/a3: r_j0 = C_0, r_jk = max(C_k, r_j,k-1 + p_j,k-1) (R3); R_k =
            // min over unscheduled j (R5); Q_l = min_j q_jl, q_jl = sum_{i>l}
            // p_ji (R4); L_k = sum_j p_jk closes the difference walk.
            // TM variants keep Q and L as packed 16-bit machine pairs (all values
            // are < 2^15, host-checked): tails q_jl come from a per-job table of
            // machine pairs (one VIMNMX.U16x2 per pair) and p_jl from another
            // (one add per pair), next to PTM in shared memory
            if constexpr (!SPARSE && EXACT && S16) {
                if (a.jp && (a.dbg_skip & 4)) continue; // diagnostics: C pass only
                if (a.jp) { // rows a2/a3 by job pairs (jp_heads), then the TMEM stores
#pragma unroll
                    for (int k = 0; k < MAXM; ++k) C[k] &= 0xffff; // the 16-bit C pass's garbage
                    const bool bd = (a.cin || !FSP_JP_LC || MAXM <= 5) ? jp_heads<MAXM, HM, NPLP, UL, TM, TN, false>(
                                                a, s_pq, Uw, urow, useg, lane, q, C, Lp, tbase,
                                                reinterpret_cast<uint16_t *>(Rs), n, node < pool ? n - d : 0)
                                          : jp_heads<MAXM, HM, NPLP, UL, TM, TN, true>(
                                                a, s_pq, Uw, urow, useg, lane, q, C, Lp, tbase,
                                                reinterpret_cast<uint16_t *>(Rs), n, node < pool ? n - d : 0);
                    if (bd) bad = true;
                    continue;
                }
            }
            int R[MAXM], Q[MAXM], Ld[MAXM];
            uint32_t Q2[HM], L2[HM], R2[HM];
#pragma unroll
            for (int k = 0; k < MAXM; ++k) {
                R[k] = INT_MAX;
                Q[k] = INT_MAX;
                Ld[k] = 0;
            }
#pragma unroll
            for (int kp = 0; kp < HM; ++kp) {
                Q2[kp] = R2[kp] = 0xffffffffu;
                L2[kp] = 0;
            }
            int cnt = 0;
            // a2/a3 for job j if it is unscheduled in this lane's node q
            auto visit = [&](int j, bool act) {
                if (act) {
                    ++cnt;
                    const int4 *pr = reinterpret_cast<const int4 *>(s_ptm + j * a.mp4);
                    int p[MAXM];
#pragma unroll
                    for (int k4 = 0; k4 < (MAXM + 3) / 4; ++k4) {
                        const int4 v = 4 * k4 < m ? pr[k4] : make_int4(0, 0, 0, 0);
                        if (4 * k4 + 0 < MAXM) p[4 * k4 + 0] = v.x;
                        if (4 * k4 + 1 < MAXM) p[4 * k4 + 1] = v.y;
                        if (4 * k4 + 2 < MAXM) p[4 * k4 + 2] = v.z;
                        if (4 * k4 + 3 < MAXM) p[4 * k4 + 3] = v.w;
                    }
                    if constexpr (TM) {
                        // heads of two machines packed by one FMA-pipe IMAD, one
                        // VIMNMX.U16x2 per pair (values < 2^16, host-checked)
                        int r = C[0];
#pragma unroll
                        for (int kp = 0; kp < HM; ++kp) {
                            const int r0 = r;
                            int r1 = r0;
                            if (2 * kp + 1 < MAXM) r1 = max(C[2 * kp + 1], r0 + p[2 * kp]);
                            if (2 * kp + 2 < MAXM) r = max(C[2 * kp + 2], r1 + p[2 * kp + 1]);
                            R2[kp] = __vminu2(R2[kp], (uint32_t)r1 * 65536u + (uint32_t)r0);
                        }
                    } else {
                        int r = C[0];
                        R[0] = min(R[0], r);
#pragma unroll
                        for (int k = 1; k < MAXM; ++k) {
                            if (k < m) {
                                r = max(C[k], r + p[k - 1]);
                                R[k] = min(R[k], r);
                            }
                        }
                    }
                    if constexpr (TM) {
                        const uint4 *pq = reinterpret_cast<const uint4 *>(s_pq + j * 2 * HMP);
#pragma unroll
                        for (int c4 = 0; c4 < HMP / 4; ++c4) {
                            const uint4 pv = pq[c4], qv = pq[HMP / 4 + c4];
                            const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w}, qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                if (4 * c4 + t < HM) {
                                    Q2[4 * c4 + t] = __vminu2(Q2[4 * c4 + t], qw[t]);
                                    L2[4 * c4 + t] += pw[t];
                                }
                            }
                        }
                    } else {
                        int qq = 0;
#pragma unroll
                        for (int l = MAXM - 1; l >= 0; --l) {
                            if (l < m) {
                                Q[l] = min(Q[l], qq);
                                qq += p[l];
                                Ld[l] += p[l];
                            }
                        }
                    }
                }
            };
            if constexpr (SPARSE) {
                // only the warp's live jobs (unscheduled in some node of the
                // warp): deep B&B blocks have a few dozen of n
                for (int w0 = 0; w0 * 32 < n; ++w0) {
                    uint32_t bits = __shfl_sync(0xffffffffu, livew, w0);
                    while (bits) {
                        const int j = w0 * 32 + __ffs(bits) - 1;
                        bits &= bits - 1;
                        const uint32_t uj = Uw[j * urow + useg + UL::word(lane, q)];
                        visit(j, (uj >> UL::bit(lane, q)) & 1u);
                    }
                }
            } else {
                for (int j = 0; j < n; ++j) {
                    const uint32_t uj = Uw[j * urow + useg + UL::word(lane, q)];
                    const bool act = (uj >> UL::bit(lane, q)) & 1u;
                    if constexpr (UL::NIB) {
                        if (!__any_sync(0xffffffffu, act)) continue; // scheduled everywhere
                    } else {
                        if (uj == 0) continue; // scheduled in every node of this half-warp
                    }
                    visit(j, act);
                }
            }
            if (node < pool && cnt != n - d) bad = true; // repeated / bad job
            if (cnt == 0) { // R6: complete schedule
#pragma unroll
                for (int k = 0; k < MAXM; ++k) {
                    R[k] = C[k];
                    Q[k] = 0;
                    Ld[k] = 0;
                }
#pragma unroll
                for (int kp = 0; kp < HM; ++kp) {
                    Q2[kp] = 0;
                    L2[kp] = 0;
                    R2[kp] = (uint32_t)C[2 * kp] | ((2 * kp + 1 < MAXM ? (uint32_t)C[2 * kp + 1] : 0u) << 16);
                }
            }
            if constexpr (TM) {
#pragma unroll
                for (int kp = 0; kp < HM; ++kp) {
                    const int k0 = 2 * kp, k1 = 2 * kp + 1 < MAXM ? 2 * kp + 1 : 2 * kp;
                    auto pk = [](int lo, int hi) { return ((uint32_t)lo & 0xffffu) | ((uint32_t)hi << 16); };
                    (void)pk;
                    (void)k0;
                    (void)k1;
                    tm_st1(tbase + (0 * HM + kp) * NPLP + q, R2[kp]);
                    tm_st1(tbase + (1 * HM + kp) * NPLP + q, R2[kp] + L2[kp]); // A = R + L
                    tm_st1(tbase + (2 * HM + kp) * NPLP + q, Q2[kp]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < MAXM; ++k) {
                    if (k < m) {
                        Rs[k * TN + q * 32 + lane] = (rt_t)R[k];
                        As[k * TN + q * 32 + lane] = (rt_t)(R[k] + Ld[k]);
                        Qs[k * TN + q * 32 + lane] = (rt_t)Q[k];
                    }
                }
            }
        }
        if (bad) atomicOr(a.err, 1);
        if constexpr (TM) tm_wait_st();
        __syncwarp();
        mark(PR_HEADS);

        // ---------------- a4/a5: couple walks (Fig. 3 lines 03-19) ----------------
        int lb[NPL]; // R1: the max over couples starts at 0
#pragma unroll
        for (int q = 0; q < NPL; ++q) lb[q] = 0;
        const bool ascending = resident == 0;
        int kc = -1, rkv[NPL], akv[NPL]; // SPARSE TM: R_k - D and A_k of the last first machine
#pragma unroll
        for (int q = 0; q < NPL; ++q) rkv[q] = akv[q] = 0;
        for (int gi = 0; gi < a.groups; ++gi) {
            const int g = dbuf ? gi : ascending ? gi : a.groups - 1 - gi;
            const long long sq = it * a.groups + gi;
            const uint8_t *tab = s_tab;
            mark(PR_WALK);
            if constexpr (RG) {
                tab = a.tables + (size_t)g * a.L.group_bytes;
            } else if (dbuf) { // wait for this group's buffer; no CTA-wide barrier
                const int b = (int)(sq % NB);
                mbar_wait(s_bar + b, (uint32_t)((sq / NB) & 1), a.wait_ns);
                __syncwarp(); // reconverged before the .sync.aligned TMEM loads
                tab = s_tab + (size_t)b * a.L.group_bytes;
            } else if (g != resident) {
                __syncthreads(); // every warp is done with the resident group
                if (threadIdx.x == 0) {
                    fence_proxy_async();
                    const uint32_t gb = group_blob(g);
                    mbar_expect_tx(s_bar, gb);
                    bulk_copy(s_tab, a.tables + (size_t)g * a.L.group_bytes, gb, s_bar);
                }
                mbar_wait(s_bar, phase);
                phase ^= 1;
                resident = g;
            }
            mark(PR_WAIT);
            if (anyvalid != 0) {
            const uint32_t *kl = reinterpret_cast<const uint32_t *>(tab);
            const uint4 *recs = reinterpret_cast<const uint4 *>(tab + a.L.kl_bytes);
            const int np = group_size(g);
            const int n2 = a.nrec >> 1, n4 = a.nrec >> 2;
            for (int pl = slice; pl < ((a.dbg_skip & 2) ? 0 : np); pl += split) {
                const uint32_t kv = kl[pl];
                const int k = kv & 0xffff, l = kv >> 16;
                // lines 06-07: timeOnM1 / timeOnM2 start at the RM minima, so
                // e = t2 - t1 starts at R_l - R_k (>= 0)
                int ee[NPL], fin[NPL]; // SPARSE TM: fin = A_k + Q_l (lines 18-19)
                if constexpr (TM && (SPARSE || KC)) {
                    // short walks (B&B blocks): one TMEM round trip per couple,
                    // R_k and A_k reloaded only when k changes ((k, l) order)
                    uint32_t rl[NPLP], ql[NPLP];
                    tm_ld<NPLP>(tbase + (0 * HM + (l >> 1)) * NPLP, rl);
                    tm_ld<NPLP>(tbase + (2 * HM + (l >> 1)) * NPLP, ql);
                    if (k != kc) {
                        uint32_t rk[NPLP], ak[NPLP];
                        tm_ld<NPLP>(tbase + (0 * HM + (k >> 1)) * NPLP, rk);
                        tm_ld<NPLP>(tbase + (1 * HM + (k >> 1)) * NPLP, ak);
                        tm_wait_ld<NPLP>(rk, ak);
#pragma unroll
                        for (int q = 0; q < NPL; ++q) {
                            rkv[q] = tm_half(rk[q], k & 1) - woff;
                            akv[q] = tm_half(ak[q], k & 1);
                        }
                        kc = k;
                    }
                    tm_wait_ld<NPLP>(rl, ql);
#pragma unroll
                    for (int q = 0; q < NPL; ++q) {
                        ee[q] = tm_half(rl[q], l & 1) - rkv[q];
                        fin[q] = akv[q] + tm_half(ql[q], l & 1);
                    }
                } else if constexpr (TM) {
                    uint32_t rl[NPLP], rk[NPLP];
                    tm_ld<NPLP>(tbase + (0 * HM + (l >> 1)) * NPLP, rl);
                    tm_ld<NPLP>(tbase + (0 * HM + (k >> 1)) * NPLP, rk);
                    tm_wait_ld<NPLP>(rl, rk);
#pragma unroll
                    for (int q = 0; q < NPL; ++q) ee[q] = tm_half(rl[q], l & 1) - tm_half(rk[q], k & 1) + woff;
                } else {
#pragma unroll
                    for (int q = 0; q < NPL; ++q)
                        ee[q] = (int)Rs[l * TN + q * 32 + lane] - (int)Rs[k * TN + q * 32 + lane] + woff;
                }
                const uint4 *rp = recs + (size_t)pl * n2;
                int n4c = n4;
                if constexpr (SPARSE) {
                    if (compact) {
                        // keep the records whose job is live, in JM order
                        const uint2 *col = reinterpret_cast<const uint2 *>(rp);
                        // four 32-position chunks per round: loads, live tests and
                        // ballots of a round are independent; only the stores
                        // depend on the running count
                        int cnt = 0;
                        const uint32_t lt = (1u << lane) - 1u;
                        if (inv) {
                            // <= 32 live jobs: lane t takes live job jt, reads its
                            // position in this couple's JM order from the inverse
                            // table, ranks it among the live positions (live-count
                            // shuffles) and stores its record at that rank
                            const int key = lane < live ? (int)(tab + a.L.pos_off)[pl * n + jt] : 0x7fffffff;
                            int rank = 0;
                            for (int u = 0; u < live; ++u) rank += __shfl_sync(0xffffffffu, key, u) < key;
                            if (lane < live) s_list[rank] = col[key];
                            cnt = live;
                        } else
                        for (int i0 = 0; i0 < a.nrec; i0 += 128) {
                            uint2 r[4];
                            uint32_t bal[4];
                            bool lv[4];
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const int i = i0 + 32 * c + lane;
                                r[c] = i < a.nrec ? col[i] : make_uint2(0u, 0u);
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                // s16 records carry the job in the top half of c1
                                // (the walk's 16x2 ops ignore that half)
                                const uint32_t j = r[c].x >> 16;
                                const uint32_t word = __shfl_sync(0xffffffffu, livew, (j >> 5) & 31);
                                lv[c] = i0 + 32 * c + lane < a.nrec && ((word >> (j & 31)) & 1u);
                                bal[c] = __ballot_sync(0xffffffffu, lv[c]);
                            }
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                if (lv[c]) s_list[cnt + __popc(bal[c] & lt)] = r[c];
                                cnt += __popc(bal[c]);
                            }
                        }
                        // pad to a whole step + the look-ahead slack with no-op records
                        const uint2 dummy = reinterpret_cast<const uint2 *>(recs)[(size_t)np * a.nrec];
                        const int cnt4 = (cnt + 3) & ~3;
                        for (int t = cnt + lane; t < cnt4 + FSP_REC_SLACK; t += 32) s_list[t] = dummy;
                        __syncwarp();
                        rp = reinterpret_cast<const uint4 *>(s_list);
                        n4c = cnt4 >> 2;
                    }
                }
                // lines 08-17, software-pipelined 4 positions per step: records
                // two steps ahead, U masks one step ahead (the group blob ends
                // with padding records so the look-ahead stays in bounds).
                // X/Y register sets alternate so no copies are needed.
                uint4 xa = rp[0], xb = rp[1]; // step 0
                uint4 ya = rp[2], yb = rp[3]; // step 1
                Mask<MW> mx0 = FSP_MASK(xa.y), mx1 = FSP_MASK(xa.w);
                Mask<MW> mx2 = FSP_MASK(xb.y), mx3 = FSP_MASK(xb.w);
                int s = 0;
#pragma unroll kUnroll
                for (; s + 2 <= n4c; s += 2) {
                    const Mask<MW> my0 = FSP_MASK(ya.y), my1 = FSP_MASK(ya.w);
                    const Mask<MW> my2 = FSP_MASK(yb.y), my3 = FSP_MASK(yb.w);
                    FSP_UPD(mx0, xa.x, xa.y);
                    FSP_UPD(mx1, xa.z, xa.w);
                    FSP_UPD(mx2, xb.x, xb.y);
                    FSP_UPD(mx3, xb.z, xb.w);
                    xa = rp[2 * s + 4];
                    xb = rp[2 * s + 5];
                    mx0 = FSP_MASK(xa.y);
                    mx1 = FSP_MASK(xa.w);
                    mx2 = FSP_MASK(xb.y);
                    mx3 = FSP_MASK(xb.w);
                    FSP_UPD(my0, ya.x, ya.y);
                    FSP_UPD(my1, ya.z, ya.w);
                    FSP_UPD(my2, yb.x, yb.y);
                    FSP_UPD(my3, yb.z, yb.w);
                    ya = rp[2 * s + 6];
                    yb = rp[2 * s + 7];
                }
                if (s < n4c) { // odd number of steps: the last one is in X
                    FSP_UPD(mx0, xa.x, xa.y);
                    FSP_UPD(mx1, xa.z, xa.w);
                    FSP_UPD(mx2, xb.x, xb.y);
                    FSP_UPD(mx3, xb.z, xb.w);
                }
                if constexpr (S16) {
#pragma unroll
                    for (int q = 0; q < NPL; ++q) ee[q] = (int)(ee[q] & 0xffff) - woff;
                }
                // lines 18-19: timeOnM2 = t1 + e with t1 = R_k + L_k at the end
                if constexpr (TM && (SPARSE || KC)) {
#pragma unroll
                    for (int q = 0; q < NPL; ++q) lb[q] = max(lb[q], ee[q] + fin[q]);
                } else if constexpr (TM) {
                    uint32_t ak[NPLP], ql[NPLP];
                    tm_ld<NPLP>(tbase + (1 * HM + (k >> 1)) * NPLP, ak);
                    tm_ld<NPLP>(tbase + (2 * HM + (l >> 1)) * NPLP, ql);
                    tm_wait_ld<NPLP>(ak, ql);
#pragma unroll
                    for (int q = 0; q < NPL; ++q)
                        lb[q] = max(lb[q], ee[q] + tm_half(ak[q], k & 1) + tm_half(ql[q], l & 1));
                } else {
#pragma unroll
                    for (int q = 0; q < NPL; ++q)
                        lb[q] = max(lb[q], ee[q] + As[k * TN + q * 32 + lane] + Qs[l * TN + q * 32 + lane]);
                }
                if constexpr (SPARSE)
                    if (compact) __syncwarp(); // the next couple rewrites s_list
            }
            } // anyvalid
            mark(PR_WALK);
            if (!RG && dbuf) {
                // release the buffer; the last of the W warps (its (sq>>1)-th
                // round of W arrivals completes) refills it with group sq + 2
                __syncwarp();
                if (lane == 0) {
                    const int b = (int)(sq % NB);
                    // release this warp's reads of the buffer (mbarrier arrive); the
                    // counter only elects the refilling warp, which then waits on the
                    // "released" mbarrier (acquire) before the TMA overwrites it
                    mbar_arrive(s_emp + b);
                    const uint32_t old = atomicAdd(&s_cnt[b], 1u);
                    if (old == (uint32_t)((sq / NB + 1) * W - 1) && sq + NB < nseq) {
                        mbar_wait(s_emp + b, (uint32_t)((sq / NB) & 1));
                        const int gn = (int)((sq + NB) % a.groups);
                        const uint32_t gb = group_blob(gn);
                        fence_proxy_async();
                        mbar_expect_tx(s_bar + b, gb);
                        bulk_copy(s_tab + (size_t)b * a.L.group_bytes,
                                  a.tables + (size_t)gn * a.L.group_bytes, gb, s_bar + b);
                    }
                }
                __syncwarp(); // lane 0 may have waited on "released": reconverge
            }
            mark(PR_RELEASE);
        }
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const long long node = tile * TN + sidx[q];
            if (node < pool) {
                if (split == 1) a.lb_out[node] = lb[q];
                else atomicMax(&a.lb_out[node], lb[q]);
            }
        }
        __syncwarp();
        mark(PR_STORE);
    }

    if constexpr (TM) { // every warp is done with its columns
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (warp == 0) tm_dealloc(*s_tm, a.tm_cols);
    }
}

template <int MAXM, bool EXACT, bool S16, int NPL, bool SPARSE, bool BYTE = true>
int launch(const fsp_lb_plan &pl, const LbArgs &a, cudaStream_t s)
{
    if constexpr (MAXM == 20 && EXACT && S16 && NPL == 4 && BYTE) {
        if (pl.recs_global) {
            lb_kernel<20, true, true, 4, SPARSE, true, true><<<pl.grid, pl.warps * 32, pl.smem_bytes, s>>>(a);
            cudaError_t e = cudaGetLastError();
            return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "lb_kernel launch");
        }
        if constexpr (!SPARSE) {
            if (pl.kcache) {
                lb_kernel<20, true, true, 4, false, true, false, true>
                    <<<pl.grid, pl.warps * 32, pl.smem_bytes, s>>>(a);
                cudaError_t e = cudaGetLastError();
                return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "lb_kernel launch");
            }
        }
    }
    lb_kernel<MAXM, EXACT, S16, NPL, SPARSE, BYTE><<<pl.grid, pl.warps * 32, pl.smem_bytes, s>>>(a);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? FSP_OK : fsp_cuda_fail(e, "lb_kernel launch");
}

template <int MAXM, bool EXACT, bool S16, int NPL, bool SPARSE, bool BYTE = true>
int configure(fsp_lb_plan &pl)
{
    // the attribute is per kernel variant and shared by every instance: set it
    // to the device's opt-in maximum, never to this plan's size
    cudaError_t e = cudaFuncSetAttribute(lb_kernel<MAXM, EXACT, S16, NPL, SPARSE, BYTE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pl.smem_optin);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "cudaFuncSetAttribute");
    if constexpr (MAXM == 20 && EXACT && S16 && NPL == 4 && BYTE) {
        e = cudaFuncSetAttribute(lb_kernel<20, true, true, 4, SPARSE, true, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem_optin);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "cudaFuncSetAttribute");
        if constexpr (!SPARSE) {
            e = cudaFuncSetAttribute(lb_kernel<20, true, true, 4, false, true, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem_optin);
            if (e != cudaSuccess) return fsp_cuda_fail(e, "cudaFuncSetAttribute");
        }
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lb_kernel<MAXM, EXACT, S16, NPL, SPARSE, BYTE>,
                                                      pl.warps * 32, pl.smem_bytes);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "occupancy");
    if (per_sm < 1) return fsp_fail(FSP_ERANGE, "lb kernel does not fit on an SM");
    pl.ctas_per_sm = per_sm;
    pl.grid = pl.num_sms * per_sm;
    return FSP_OK;
}

// (MAXM, EXACT, S16, NPL, SPARSE) specialisations: exact m for Taillard's
// 5/10/20 machines (2 or 4 nodes per lane, dense or sparse walk), generic m
// with 2 nodes per lane and the dense walk.
#define FSP_EXACT_CASE(M, FN, S, ...)                                           \
    case M * 2 + 1:                                                             \
        if (pl.sparse)                                                          \
            return pl.npl == 4 ? FN<M, true, S, 4, true>(__VA_ARGS__)           \
                               : FN<M, true, S, 2, true>(__VA_ARGS__);          \
        if (!pl.byte_rows)                                                      \
            return pl.npl == 4 ? FN<M, true, S, 4, false, false>(__VA_ARGS__)   \
                               : FN<M, true, S, 2, false, false>(__VA_ARGS__);  \
        return pl.npl == 4 ? FN<M, true, S, 4, false>(__VA_ARGS__)              \
                           : FN<M, true, S, 2, false>(__VA_ARGS__);
#define FSP_DISPATCH_M(FN, S, ...)                                              \
    switch (pl.maxm * 2 + (pl.exact ? 1 : 0)) {                                 \
        FSP_EXACT_CASE(5, FN, S, __VA_ARGS__)                                   \
        FSP_EXACT_CASE(10, FN, S, __VA_ARGS__)                                  \
        FSP_EXACT_CASE(20, FN, S, __VA_ARGS__)                                  \
    case 8 * 2: return FN<8, false, S, 2, false>(__VA_ARGS__);                  \
    case 16 * 2: return FN<16, false, S, 2, false>(__VA_ARGS__);                \
    case 24 * 2: return FN<24, false, S, 2, false>(__VA_ARGS__);                \
    default: return FN<32, false, S, 2, false>(__VA_ARGS__);                    \
    }
#define FSP_DISPATCH(FN, ...)                                                   \
    if (pl.s16) {                                                               \
        FSP_DISPATCH_M(FN, true, __VA_ARGS__)                                   \
    } else {                                                                    \
        FSP_DISPATCH_M(FN, false, __VA_ARGS__)                                  \
    }

} // namespace

static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Set the kernel variant's dynamic-smem attribute and fill ctas_per_sm / grid.
static int occupancy_of(fsp_lb_plan &pl)
{
    FSP_DISPATCH(configure, pl);
    return FSP_OK;
}

// couple-group buffers per CTA when the couples take several groups
// (FSP_LB_DBUF: 0/1 = one buffer + CTA barrier, 2..FSP_MAX_GBUF = multi-buffered)
static int nbuf_want()
{
    const char *s = getenv("FSP_LB_DBUF");
    const int v = s ? atoi(s) : 2;
    return v <= 1 ? 1 : std::min(v, FSP_MAX_GBUF);
}

// Choose the machine specialisation, warps per CTA and couple groups so that
// one couple group + PTM + U + per-warp scratch fit the opt-in shared memory
// and every U address fits the 16-bit record field.
int fsp_plan_lb(fsp_instance *inst, bool sparse)
{
    fsp_lb_plan &pl = sparse ? inst->plan_bb : inst->plan;
    const int n = inst->n, m = inst->m, P = inst->P;
    pl.exact = (m == 5 || m == 10 || m == 20);
    // 16-bit walk when e + D fits u16 with D = max p: 0 <= e <= t2 <= (n+m-1)*max p,
    // e + x >= -max p; R, A, Q are bounded by t2
    pl.s16 = (int64_t)(n + m) * inst->max_p <= 65535;
    if (const char *s = getenv("FSP_LB_S16")) pl.s16 = pl.s16 && atoi(s) != 0;
    // sparse walk: exact-m s16 specialisations (records carry the job id),
    // 64 <= n <= 1024 (below 64 jobs the compaction does not pay: measured)
    pl.sparse = sparse && pl.exact && pl.s16 && n >= 64 && n <= 1024;
    // placement ablation (NEXT-3): couple records read from global memory by
    // the 20-machine dense byte-row kernel (FSP_LB_RECS=global)
    {
        const char *rg = getenv(sparse ? "FSP_BB_RECS" : "FSP_LB_RECS");
        pl.recs_global = rg && std::string(rg) == "global";
    }
    if (pl.exact) pl.maxm = m;
    else if (m <= 8) pl.maxm = 8;
    else if (m <= 16) pl.maxm = 16;
    else if (m <= 24) pl.maxm = 24;
    else if (m <= 32) pl.maxm = 32;
    else return fsp_fail(FSP_ERANGE, "m too large");
    int dev = inst->device, optin = 0, sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "device attribute");
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return fsp_cuda_fail(e, "device attribute");
    pl.num_sms = sms;
    pl.smem_optin = optin;
    const int mp4 = (m + 3) & ~3;
    pl.nrec = (n + 3) & ~3; // walk steps of 4 positions
    pl.npl = 2;
    // job-pair heads (dense TMEM plans, exact m): the heads, tails and loads of
    // two jobs per 16x2 op, scheduled halves pushed above every real value by
    // the offset M: needs M > (n+m)*max p (every real r_jk, q_jl) and
    // M + sum_k p_jk <= 65535; the low halves of the packed loads collect
    // ceil(n/2)*max p (see jp_heads in lb_kernel)
    {
        int64_t maxsum = 0;
        for (int j = 0; j < n; ++j) {
            int64_t sj = 0;
            for (int k = 0; k < m; ++k) sj += inst->h_ptm[(size_t)j * m + k];
            maxsum = std::max(maxsum, sj);
        }
        const int64_t M = (65535 - maxsum) & ~int64_t(15);
        pl.jp_m = (int)std::max<int64_t>(M, 0);
        pl.jp = !sparse && pl.exact && pl.s16 && M > (int64_t)(n + m) * inst->max_p &&
                (int64_t)((n + 1) / 2) * inst->max_p <= 65535;
        if (const char *s = getenv("FSP_LB_JP")) pl.jp = pl.jp && atoi(s) != 0;
    }
    // 8-bit PTM rows for the jp plans' C pass when every p fits a byte
    pl.ptm8 = pl.jp && inst->max_p <= 255 && m <= 5;
    if (const char *s = getenv("FSP_LB_PTM8")) pl.ptm8 = pl.ptm8 && atoi(s) != 0;
    // R_k / A_k cached across couples in dense walks of short job lists (KC)
    pl.kcache = !sparse && n <= 64;
    if (const char *s = getenv("FSP_LB_KCACHE")) pl.kcache = !sparse && atoi(s) != 0;
    // Candidates: nodes per lane (4 only for the exact-m specialisations), warps
    // per CTA, fewest couple groups that fit.  Score = resident warps per SM
    // (latency hiding) x 1.5 for 4 nodes per lane (half the table and mask
    // traffic per node; +18 % measured at 200x20) / (1 + 1.5 % per extra group
    // reload).  Env FSP_LB_NPL / FSP_LB_WARPS pin a choice (sweeps, tests).
    int npl_lo = 2, npl_hi = pl.exact ? 4 : 2;
    if (const char *s = getenv("FSP_LB_NPL")) npl_lo = npl_hi = (atoi(s) == 4 && pl.exact) ? 4 : 2;
    // sparse walk: 4 nodes per lane (128-node blocks) since the difference walk and
    // TMEM heads (ta091 B&B: 390 M nodes/s vs 314 M with 64-node blocks, whose
    // smaller live sets no longer outweigh the per-node table and mask traffic)
    if (pl.sparse) npl_lo = npl_hi = getenv("FSP_BB_NPL") && atoi(getenv("FSP_BB_NPL")) == 2 ? 2 : 4;
    int w_lo = 1, w_hi = pl.maxm > 20 ? 8 : pl.maxm <= 5 ? 4 : 16; // = the kernel's launch bounds
    if (const char *s = getenv(sparse ? "FSP_BB_WARPS" : "FSP_LB_WARPS")) w_lo = w_hi = std::max(1, std::min(w_hi, atoi(s)));
    double best = -1.0;
    fsp_lb_plan bestp = pl;
    for (int npl = npl_lo; npl <= npl_hi; npl += 2) {
        for (int lay = 0; lay < 2; ++lay) // 0: byte rows, 1: nibble rows (m >= 10, not sparse)
        for (int W = w_hi; W >= w_lo; --W) {
            if (lay == 1 && !(pl.s16 && pl.maxm >= 10 && pl.exact && !pl.sparse)) break;
            if (const char *e = getenv("FSP_LB_ROWS")) // experiments: 0 = byte, 1 = nibble
                if (atoi(e) != lay && pl.s16 && pl.maxm >= 10 && pl.exact && !pl.sparse) break;
            // warps are dealt to the 4 SMSPs by id % 4: a W that is not a multiple
            // of 4 leaves some SMSPs with an extra warp that paces the whole CTA
            // (measured: 200x20, 10 warps 120 M/s vs 12 warps 140 M/s)
            if (W % 4 != 0 && w_lo != w_hi) continue;
            // sparse-plan rows are padded by npl words so the per-job rows of
            // one warp spread over the banks (building U touches 32 different
            // jobs at once; it dominates for deep B&B nodes, not for D1 pools)
            // s16: nibble rows (one word per lane, ceil(32/LPW) words per warp);
            // made odd so the 32 jobs a warp clears at once hit 32 banks
            const bool nib = pl.s16 && pl.maxm >= 10; // = ULayout::NIB
            // = ULayout::WPR: byte rows 8 words (32 lanes x 8 bits), nibble rows
            // ceil(32 / lanes per word)
            const int wpr = !nib ? npl : lay == 0 ? 8 : (32 + 31 / (npl + 1) - 1) / (31 / (npl + 1));
            // nibble: per-warp blocks of (n+1) rows of wpr|1 words (odd: the 32 jobs a
            // warp clears at once hit 32 banks); record offsets j*4*urow < 64 KB
            // (FSP_LB_UROW_PAD=0: byte rows unpadded, 8 words; measured below)
            const bool pad = !getenv("FSP_LB_UROW_PAD") || atoi(getenv("FSP_LB_UROW_PAD")) != 0;
            const int urow = nib ? (lay == 0 && !pad ? wpr : wpr | 1) : npl * W;
            if (!nib && (size_t)(n + 1) * 4 * urow > 65535) continue; // 16-bit U row offsets
            if (nib && (size_t)(n + 1) * 4 * urow > 65535) continue;
            fsp_lb_layout L{};
            L.urow_words = urow;
            L.u_bytes = align16((size_t)(nib ? W : 1) * (n + 1) * 4 * urow);
            L.off_u = 0;
            // + the packed (p, q) machine-pair rows of the TM (nibble) variants
            // jp plans: + the job-pair rows [ceil(n/2)][mp4] (p_2i,k | p_2i+1,k << 16)
            // (every TMA bulk copy is a multiple of 16 bytes: the row block is padded)
            L.ptm_bytes = pl.jp ? align16((size_t)n * fsp_ptm_row_words(true, pl.ptm8, m) * 4) + (size_t)((n + 1) / 2) * mp4 * 4
                                : align16((size_t)n * mp4 * 4) + (nib ? (size_t)n * fsp_pq_words(pl.maxm) * 4 : 0);
            L.off_ptm = L.u_bytes;
            L.off_bar = L.off_ptm + L.ptm_bytes;
            // nibble variants keep R/A/Q in TMEM: ceil(W/4) blocks of 3*ceil(maxm/2)*npl
            // columns per lane quarter, allocated as a power of two >= 32 per CTA
            int tm_cols = 0;
            if (nib) {
                const int need = (W + 3) / 4 * 3 * ((pl.maxm + 1) / 2) * npl;
                tm_cols = 32;
                while (tm_cols < need) tm_cols *= 2;
                if (tm_cols > 512) continue;
            }
            L.rt_bytes = nib ? 0 : 3 * (size_t)pl.maxm * 32 * npl * (pl.s16 ? 2 : 4);
            L.off_rt = L.off_bar + 32 * FSP_MAX_GBUF; // mbarriers, counters, TMEM address
            L.list_bytes = pl.sparse ? align16(((size_t)pl.nrec + FSP_REC_SLACK + 4) * 8) : 0;
            L.off_list = align16(L.off_rt + (size_t)W * L.rt_bytes);
            L.off_tab = align16(L.off_list + (size_t)W * L.list_bytes);
            for (int G = 1; G <= P; ++G) {
                const int ppg = (P + G - 1) / G;
                const int Greal = (P + ppg - 1) / ppg;
                L.kl_bytes = align16((size_t)ppg * 4);
                // + FSP_REC_SLACK padding records for the walk's look-ahead
                size_t gb = align16(L.kl_bytes +
                                    ((size_t)ppg * pl.nrec + FSP_REC_SLACK) * sizeof(fsp_rec));
                // sparse plan, n <= 256: + the inverse position table (u8
                // [couple][job] = position of the job in the couple's JM order)
                L.pos_off = 0;
                if (pl.sparse && n <= 256 && !getenv("FSP_BB_NOINV")) {
                    L.pos_off = gb;
                    gb = align16(gb + (size_t)ppg * n);
                }
                // two or more groups: double-buffered (two group buffers) unless
                // FSP_LB_DBUF=0 (one buffer, CTA barrier per group switch)
                const int nb = Greal > 1 ? std::min(Greal, nbuf_want()) : 1;
                const bool db = nb >= 2;
                if (L.off_tab + nb * gb <= (size_t)optin) {
                    fsp_lb_plan c = pl;
                    L.group_bytes = gb;
                    c.L = L;
                    c.npl = npl;
                    c.groups = Greal;
                    c.pairs_per_group = ppg;
                    c.warps = W;
                    c.smem_bytes = L.off_tab + nb * gb;
                    c.dbuf = db ? nb : 0;
                    c.tm_cols = tm_cols;
                    c.byte_rows = lay == 0;
                    // co-resident CTAs must fit the SM's 512 TMEM columns (an
                    // allocation beyond them would wait for another CTA to exit)
                    if (occupancy_of(c) == FSP_OK && c.ctas_per_sm > 0 &&
                        c.ctas_per_sm * tm_cols <= 512) {
                        // byte rows: one FMA op less per position and the fused
                        // lane ingest (+11 % at 200x20; 500x20: 8 warps of byte
                        // rows 14.6 ms vs 12 warps of nibble rows 15.3 ms)
                        const double score = (double)W * c.ctas_per_sm * (npl == 4 ? 1.5 : 1.0) *
                                             (nib && lay == 0 ? 1.25 : 1.0) /
                                             (1.0 + (db ? 0.005 : 0.015) * (Greal - 1));
                        if (score > best) {
                            best = score;
                            bestp = c;
                        }
                    }
                    break; // more groups only cost for this (npl, W)
                }
                if (ppg == 1) break;
            }
        }
    }
    if (best > 0) {
        pl = bestp;
        return occupancy_of(pl); // sets the attribute for the chosen variant
    }
    return fsp_fail(FSP_ERANGE, "instance tables do not fit in shared memory");
}

// Couple split for pools with fewer tiles than warp slots (latency-bound
// otherwise: a 4,096-node pool is 32 tiles on 148 x 16 warps); the pool size
// of a device-sized launch (B&B) is only bounded by `pool`.
int fsp_lb_split(const fsp_lb_plan &pl, int64_t pool)
{
    int split = 1;
    const int64_t tiles = (pool + 32 * pl.npl - 1) / (32 * pl.npl);
    const int64_t slots = (int64_t)pl.grid * pl.warps;
    while (split < pl.warps && tiles * split * 2 <= slots) split *= 2;
    if (const char *e = getenv("FSP_LB_SPLIT")) { // experiments and tests: a power of two
        const int v = std::max(1, std::min(pl.warps, atoi(e)));
        for (split = 1; split * 2 <= v;) split *= 2;
    }
    while (pl.warps % split) split /= 2;
    return split;
}

// First node of the last tile iteration of an unsplit launch.
int64_t fsp_lb_tail_first(const fsp_lb_plan &pl, int64_t pool)
{
    const int64_t tn = 32 * pl.npl, tiles = (pool + tn - 1) / tn;
    const int64_t slots = (int64_t)pl.grid * pl.warps;
    const int64_t niter = (tiles + slots - 1) / slots;
    return niter > 0 ? (niter - 1) * slots * tn : 0;
}

// Split of the last tile iteration of an unsplit launch: the tiles left for
// it are spread over up to all warp slots (couple split, atomicMax combine).
int fsp_lb_tail_split(const fsp_lb_plan &pl, int64_t pool, int split)
{
    // measured on 200x20 1M pools: the idle warps of the partial wave were the
    // whole 8 % "wait" share; splitting their tiles (repeated phase A) did not
    // shorten the round-2 launch (5.80 vs 5.82 ms), but with phase A at ~20 %
    // it does (round 2b, profiles/r02/tail_split_ab.txt: 4.85 -> 4.80 ms,
    // 50x20 1.384 -> 1.364): on unless FSP_LB_TAIL=0
    if (split != 1 || pool <= 0) return 1;
    if (getenv("FSP_LB_TAIL") && atoi(getenv("FSP_LB_TAIL")) == 0) return 1;
    const int64_t tn = 32 * pl.npl, tiles = (pool + tn - 1) / tn;
    const int64_t slots = (int64_t)pl.grid * pl.warps;
    const int64_t rem = tiles - (fsp_lb_tail_first(pl, pool) / tn);
    int s = 1;
    while (s < pl.warps && rem * s * 2 <= slots) s *= 2;
    while (pl.warps % s) s /= 2;
    return s;
}

int fsp_launch_lb(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                  const int32_t *depth, int64_t pool, int32_t *lb_out, cudaStream_t s)
{
    if (inst->wpn) return fsp_launch_lb_wpn(inst, prefix, stride, depth, pool, lb_out, s);
    return fsp_launch_lb_dev(inst, prefix, stride, depth, pool, nullptr, nullptr, 0, false, lb_out, s,
                             0);
}

int fsp_launch_lb_dev(const fsp_instance *inst, const uint16_t *prefix, int32_t stride,
                      const int32_t *depth, int64_t pool, const int64_t *pool_dev,
                      const int32_t *cin, int32_t cin_stride, bool sparse, int32_t *lb_out,
                      cudaStream_t s, int grid_limit, const uint16_t *ulist)
{
    fsp_lb_plan pl = sparse ? inst->plan_bb : inst->plan;
    // host path: a few SMs are left to the PCIe gather kernel of the next chunk
    if (grid_limit > 0 && grid_limit < pl.grid) pl.grid = grid_limit;
    const uint8_t *tables = sparse ? inst->d_tables_bb : inst->d_tables;
    LbArgs a;
    a.tables = tables;
    a.ptm = sparse ? inst->d_ptm32s_bb : inst->d_ptm32s;
    a.jp = pl.jp ? 1 : 0;
    a.sort_depth = getenv("FSP_LB_SORT") ? atoi(getenv("FSP_LB_SORT")) : 1;
    a.prow = fsp_ptm_row_words(pl.jp, pl.ptm8, inst->m);
    a.jp_off = (int)(align16((size_t)inst->n * a.prow * 4) / 4); // words to the jp / pq rows
    for (int kp = 0; kp < 16; ++kp) {
        uint32_t lo = 0, hi = 0;
        for (int j = 0; pl.jp && j < inst->n; ++j) {
            if (2 * kp < inst->m) lo += (uint32_t)inst->h_ptm[(size_t)j * inst->m + 2 * kp];
            if (2 * kp + 1 < inst->m) hi += (uint32_t)inst->h_ptm[(size_t)j * inst->m + 2 * kp + 1];
        }
        a.ltot2[kp] = lo | (hi << 16); // each sum <= n * max p < 2^16 (the 16-bit walk's condition)
    }
    a.ptm8 = pl.jp && pl.ptm8 ? 1 : 0;
    a.jp_m = (uint32_t)pl.jp_m;
    a.one = 1u;
    a.cin = cin;
    a.cin_stride = cin_stride;
    // eight job ids per lane pay off only for long prefixes (measured: 20x5 and
    // 20x20 faster with one id per lane, 200x20 faster with eight)
    a.vec_rows = getenv("FSP_LB_VECROWS") ? atoi(getenv("FSP_LB_VECROWS")) : (inst->n >= 128);
    a.prefix = prefix;
    a.depth = depth;
    a.lb_out = lb_out;
    a.err = inst->d_err;
    a.pool = pool;
    a.pool_dev = reinterpret_cast<const long long *>(pool_dev);
    a.L = pl.L;
    a.groups = pl.groups;
    a.ppg = pl.pairs_per_group;
    a.n = inst->n;
    a.m = inst->m;
    a.P = inst->P;
    a.mp4 = (inst->m + 3) & ~3;
    a.nrec = pl.nrec;
    a.stride = stride;
    a.hi_mul = 0x10000u;
    a.tm_cols = (uint32_t)pl.tm_cols;
    a.dbuf = pl.dbuf;
    a.woff = inst->max_p;
    a.split = fsp_lb_split(pl, pool);
    a.tail_split = pool_dev ? 1 : fsp_lb_tail_split(pl, pool, a.split);
    a.wait_ns = getenv("FSP_LB_WAIT_NS") ? (uint32_t)atol(getenv("FSP_LB_WAIT_NS")) : 1000000u;
    a.dbg_skip = getenv("FSP_LB_DEBUG_SKIP") ? atoi(getenv("FSP_LB_DEBUG_SKIP")) : 0;
    a.lane_ingest = getenv("FSP_LB_LANE_INGEST") ? atoi(getenv("FSP_LB_LANE_INGEST")) : 1;
    // unscheduled lists: byte-row plans with supplied completion times only
    // (the B&B's lazy child rows rely on this: with a list, no prefix is read)
    a.ulist = ulist && cin && pl.s16 && pl.maxm >= 10 && pl.byte_rows ? ulist : nullptr;
    if (a.ulist) a.lane_ingest = 1;
    a.prof = nullptr;
    static unsigned long long *prof_buf = nullptr; // diagnostics only (FSP_LB_PROF=1)
    const bool prof = getenv("FSP_LB_PROF") && atoi(getenv("FSP_LB_PROF")) != 0;
    if (prof) {
        if (!prof_buf && cudaMalloc(&prof_buf, 8 * PR_N) != cudaSuccess) prof_buf = nullptr;
        if (prof_buf) cudaMemsetAsync(prof_buf, 0, 8 * PR_N, s);
        a.prof = prof_buf;
    }
    if (a.split > 1 && pool > 0) { // R1: every LB is a max starting at 0
        cudaError_t e = cudaMemsetAsync(lb_out, 0, sizeof(int32_t) * (size_t)pool, s);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "lb_out clear");
    } else if (a.tail_split > 1) { // only the last iteration's nodes are combined
        const int64_t first = fsp_lb_tail_first(pl, pool);
        cudaError_t e = cudaMemsetAsync(lb_out + first, 0, sizeof(int32_t) * (size_t)(pool - first), s);
        if (e != cudaSuccess) return fsp_cuda_fail(e, "lb_out clear");
    }
    const int rc = [&]() -> int { FSP_DISPATCH(launch, pl, a, s); }();
    if (prof && prof_buf && rc == FSP_OK) {
        unsigned long long h[PR_N];
        cudaMemcpyAsync(h, prof_buf, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        double tot = 0;
        for (int i = 0; i < PR_N; ++i) tot += (double)h[i];
        fprintf(stderr, "FSP_LB_PROF pool=%lld warps=%d split=%d: ingest %.1f%% heads %.1f%% wait %.1f%% "
                        "walk %.1f%% release %.1f%% store %.1f%% (%.3g warp-cycles)\n",
                (long long)pool, pl.warps, a.split, 100 * h[0] / tot, 100 * h[1] / tot, 100 * h[2] / tot,
                100 * h[3] / tot, 100 * h[4] / tot, 100 * h[5] / tot, tot);
    }
    return rc;
}
