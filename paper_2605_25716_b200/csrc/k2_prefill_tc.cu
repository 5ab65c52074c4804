// k2_prefill_tc.cu -- K2 prefill form on the 5th-generation tensor cores: keyless partial
// attention over the scrambled KV shard for many query rows (flash attention with tcgen05).
//
// Replaces shard_attention(q', K', V', none) (attention.cpp:42-78) when the delegated span has
// many rows (prefill; try_serve_q, protocol.cpp:1072-1095). The mask is always `none` for
// delegated shards. Output per split: locally normalised O' (f32) and the
// reference's (row_max, exp_sum) statistics, exactly like the decode kernel.
//
// One CTA = up to two 128-row Q tiles of one (request, q head) x one KV split -- or, for GQA
// decode ("grouped" mode), the G q heads x L_q rows of one (request, kv head), so K/V stream
// from HBM once per group instead of once per q head. With one split the CTAs are persistent
// and walk ranges of key tiles instead (stream-K, below). 12 warps (10, 11 idle; setmaxnreg):
//   warp 8      TMA producer: Q0/Q1 per segment, K_j / V_j tiles (128 keys) into rings
//   warp 9      MMA issuer (one lane): S_g = Q_g K_j^T (SS, K-major) into TMEM, and
//               O_g += P_g V_j with P_g read straight from TMEM (TS form; V as an MN-major B)
//   warps 0-3   softmax for Q tile 0, warps 4-7 for Q tile 1 (thread = row = TMEM lane):
//               tcgen05.ld S, online softmax in the log2 domain, P in bf16 written back over
//               S with tcgen05.st; lazy rescaling of O (only when the running max grows by
//               more than 2^8, FA4-style) so most tiles never touch O.
// The issue order S0(j) S1(j) PV0(j) S0(j+1) PV1(j) S1(j+1) ... ping-pongs the two softmax
// groups so the tensor pipe always has the other tile's work queued. TMEM: S0|S1|O0|O1 =
// 4 x 128 columns (P_g aliases the first 64 columns of S_g).
#include <cmath>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "tc_util.cuh"

namespace sda {

struct K2TcParams {
    int64_t q_rows;        // Lq
    int64_t kv_cap;
    const int32_t* kv_len;
    float* out_o;
    float* out_stats;
    int64_t n_batch;
    int q_heads;
    int kv_heads;
    int n_splits;
    int n_qpairs;          // ceil(Lq / 256) (normal mode)
    // causal (the inquirer's local span, AttentionMask::causal(offset), attention.hpp:25-27; split
    // mode, normal tiles only): key j is visible to span row i iff j <= i + causal_offset. The grid
    // is then x = q head, y = c < ceil(n_qpairs / 2): the CTA runs Q-tile pair n_qpairs - 1 - c (the
    // longer key range) and then pair c, so every CTA gets about the same number of key tiles
    int causal;
    int64_t causal_offset;
    int grouped;           // 1: GQA decode mode, one CTA per (request, kv head): its G = Hq/Hkv
                           //    q heads x Lq rows (contiguous in Q) form the Q tile
    float scale_log2;      // log2(e) / sqrt(d)
    // remote records (K2Params): O' / stats of request b straight into peer dest = b / b_per
    int remote;
    int64_t b_per;
    int64_t rec_stride;
    float* rec_peer[kMaxPeers];
    uint32_t* peer_flag[kMaxPeers];
    uint32_t* dest_counters;
    const uint32_t* epoch;
    // stream-K mode (one split, the caller's workspace): persistent CTAs over the linear tile
    // order, pieces of a unit merged by its last finisher through sk_buf (3 slots x 256 rows per
    // CTA) and sk_tick (one zeroed, self-resetting u32 per unit)
    int sk;
    int sk_gq;             // CTAs per group (Q-tile pairs walked in lockstep); divides n_qpairs
    float* sk_buf;
    uint32_t* sk_tick;
};

#ifdef SDA_K2_TRACE
// debug build only (tools/k2_trace.py): globaltimer stamps of CTA (0,0,0) -- [kind][j], kinds:
// 0/1 softmax g got S, 2/3 softmax g arrives with P, 4/5 PV0/PV1 issue, 6/7 MMA loop top / V ready,
// 8 before the P1 wait, 9/10 before / after the K(j+1) wait
__device__ uint64_t g_k2_trace[24][64];
__device__ uint64_t g_k2_cta[1024][2];   // every CTA's (start, end) globaltimer
__device__ __forceinline__ void k2_cta_stamp(int which) {
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && blockIdx.x < 1024) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_k2_cta[blockIdx.x][which] = t;
    }
}
#define K2_CTA_STAMP(w) k2_cta_stamp(w)
__device__ __forceinline__ void k2_stamp(int kind, int64_t j) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < 64) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_k2_trace[kind][j] = t;
    }
}
#define K2_STAMP(k, j) k2_stamp(k, j)
// the pair's rank-1 CTA (blockIdx.x == 1)
__device__ __forceinline__ void k2_stamp1(int kind, int64_t j) {
    if (blockIdx.x == 1 && blockIdx.y == 0 && blockIdx.z == 0 && j < 64) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_k2_trace[kind][j] = t;
    }
}
#define K2_STAMP1(k, j) k2_stamp1(k, j)
#else
#define K2_STAMP1(k, j)
#define K2_STAMP(k, j)
#define K2_CTA_STAMP(w)
#endif

// The MMA warp's waits for P sit on the S -> softmax -> PV -> S chain of each Q tile. A plain
// try_wait (suspending for the default time) cost ~100 ns of wake-up per hand-off against a
// test_wait spin (+2 % on C3, tools/k2_trace.py); but the spin takes issue slots from the softmax
// warps 1 and 5 on the MMA warp's SMSP, and warp 1 is the last of its group to hand P over in every
// traced tile (tools/k2_trace_warps.py). try_wait with a suspend-time hint wakes on the phase and
// leaves the slots free: C3 K2 454-457 us against 461-466 us spinning
// (profiles/k2_prefill_split_rows_r02.txt). SDA_K2_PWAIT_NS: < 0 try_wait with a |n| ns hint,
// 0 spin, > 0 spin with an n ns nanosleep between polls.
#ifndef SDA_K2_PWAIT_NS
#define SDA_K2_PWAIT_NS -1000
#endif
// the softmax warps' wait for S: try_wait, optionally with a suspend-time hint (ns)
#ifndef SDA_K2_SWAIT_NS
#define SDA_K2_SWAIT_NS 0
#endif
#if SDA_K2_SWAIT_NS > 0
#define K2_WAIT_S(b, ph) tc::mbar_wait_hint<SDA_K2_SWAIT_NS>(b, ph)
#else
#define K2_WAIT_S(b, ph) tc::mbar_wait(b, ph)
#endif
#if SDA_K2_PWAIT_NS < 0
#define K2_WAIT_P1(b, ph) tc::mbar_wait_hint<-(SDA_K2_PWAIT_NS)>(b, ph)
#elif SDA_K2_PWAIT_NS > 0
#define K2_WAIT_P1(b, ph) tc::mbar_wait_backoff<SDA_K2_PWAIT_NS>(b, ph)
#else
#define K2_WAIT_P1(b, ph) tc::mbar_wait_spin(b, ph)
#endif
// The pair form's issuers wait on barriers that rank 1's relays complete with remote arrives, which
// do not wake a suspended try_wait: they poll (SDA_K2_PAIR_PWAIT_NS > 0: with that nanosleep between
// polls). Its relay warps wait on their own CTA's barriers (SDA_K2_RELAY_HINT=1: suspend-hint
// try_wait instead of a spin).
#ifndef SDA_K2_PAIR_PWAIT_NS
#define SDA_K2_PAIR_PWAIT_NS 0
#endif
#ifndef SDA_K2_RELAY_HINT
#define SDA_K2_RELAY_HINT 1
#endif
#if SDA_K2_PAIR_PWAIT_NS > 0
#define K2_WAIT_P2(b, ph) tc::mbar_wait_backoff<SDA_K2_PAIR_PWAIT_NS>(b, ph)
#else
#define K2_WAIT_P2(b, ph) tc::mbar_wait_spin(b, ph)
#endif
#define K2_WAIT_P(b, ph)             \
    do {                             \
        if constexpr (PAIR)          \
            K2_WAIT_P2(b, ph);       \
        else                         \
            K2_WAIT_P1(b, ph);       \
    } while (0)
#if SDA_K2_RELAY_HINT
#define K2_WAIT_RELAY(b, ph) tc::mbar_wait_hint<1000>(b, ph)
#else
#define K2_WAIT_RELAY(b, ph) tc::mbar_wait_spin(b, ph)
#endif

namespace k2tc {
constexpr int D = 128;
constexpr int TILE = 128;
constexpr int TILE_BYTES = TILE * D * 2;          // 32 KB bf16 tile
constexpr int BLK = TILE * 128;                   // [128 x 64] swizzled block (16 KB)
constexpr int OFF_Q0 = 0, OFF_Q1 = OFF_Q0 + TILE_BYTES;
// P handed to the MMA in parts: part i's PV issues while the softmax exponentiates part i+1
// (C3: 1 part 476-480 us, 2 parts 460-467 us, 4 parts 531 us -- the extra waits and stores
// cost more than the overlap gains)
#ifndef SDA_K2_PPARTS
#define SDA_K2_PPARTS 2
#endif
#define SDA_K2_PSPLIT (SDA_K2_PPARTS > 1)
constexpr int kPParts = SDA_K2_PPARTS;
#ifndef SDA_K2_KSTAGES
#define SDA_K2_KSTAGES 2
#endif
constexpr int KST = SDA_K2_KSTAGES;               // K ring stages (V: 2)
constexpr int OFF_K = OFF_Q1 + TILE_BYTES;
constexpr int OFF_V = OFF_K + KST * TILE_BYTES;   // 2 stages
constexpr int OFF_BAR = OFF_V + 2 * TILE_BYTES;
// barriers: q_full, k_full[KST], k_empty[KST], v_full[2], v_empty[2], s_full[2], p_full[2],
// o_final[2], q_empty, o_empty[2], p_part[2][kPParts - 1]
constexpr int NBAR = 14 + 2 * KST + 2 * (SDA_K2_PPARTS > 1 ? SDA_K2_PPARTS - 1 : 0);
// Split rows (SDA_K2_HELP=1): each Q tile's softmax runs on two warpgroups -- the primary warps
// 0-7 take keys 0-63 of every tile (and everything else: the O rescale, the epilogue, stream-K
// merges), helper warps 12-19 keys 64-127 of the same rows (the same TMEM lanes: warp % 4). The
// per-tile chain S -> softmax -> PV -> S then carries half the exponentials per thread. The two
// halves of a row exchange their tile max (and, at a segment's end, the row sum) through shared
// memory under a 64-thread named barrier per (tile, lane quarter); the primary hands P's first
// 64 keys to the MMA on p_part, the helper the second 64 on p_full. Opt-in: parity-green but
// C3 498-501 us against 464-468 us for the default (half the logits per thread take ~90 % of the
// whole row's time: the softmax is bound by the SM's shared throughput, K2 prefill).
#ifndef SDA_K2_HELP
#define SDA_K2_HELP 0
#endif
constexpr bool kHelp = SDA_K2_HELP != 0;
static_assert(!kHelp || SDA_K2_PPARTS == 2, "split rows hand P over in two parts");
constexpr int SEG_SLOTS = kHelp ? 16 : 8;
// exchange: tile max [tile parity][primary, helper][Q tile][row], row sum [segment parity][Q tile][row]
constexpr int XCH_BYTES = kHelp ? (2 * 2 * 2 * 128 + 2 * 2 * 128) * 4 : 0;
constexpr int OFF_SEG = OFF_BAR + NBAR * 8 + 16;   // per softmax warp: segment state (SoftKeep)
constexpr int OFF_XCH = OFF_SEG + SEG_SLOTS * 128;
constexpr int SMEM = OFF_XCH + XCH_BYTES;
// The CTA-pair form (PAIR; opt-in, SDA_K2_PAIR=1 -- parity-green but 495-505 us on C3 against
// 445-454 us for the form above (second session, with the exponential mix and relay hint waits:
// 469-476 us against 448 us): with the chain decoupled both softmax groups run at once and
// each takes 1.5-1.8 us per tile instead of 1.05, so the SM's softmax throughput, not the chain,
// bounds the step): a cluster of two CTAs issues every MMA as one M = 256 tcgen05.mma
// (cta_group::2; rank 0 issues): each CTA keeps its own two Q tiles, S and O in its TMEM, and only
// HALF of every K tile (64 keys) and V tile (64 of the d columns) in its shared memory. That halves
// each SM's shared-memory operand traffic, and the room it frees holds P_g in SMEM (a SW128 K-major
// A operand) instead of over S_g in TMEM -- so S_g(j+1) goes into TMEM as soon as the softmax has
// S_g(j) in registers, and the S -> softmax -> PV -> S chain of a Q tile becomes softmax ->
// softmax. K and V half tiles share one 6-slot ring in the order the MMAs consume them (K(j+1) for
// S(j+1), then V(j) for PV(j)). (One CTA with P in SMEM was measured SMEM-bound: DESIGN.md.)
template <bool PAIR>
struct Lay {
    static constexpr int KST = PAIR ? 6 : k2tc::KST;                      // K ring (PAIR: K/V half-tile ring)
    static constexpr int SLOT = PAIR ? TILE_BYTES / 2 : TILE_BYTES;
    static constexpr int OFF_P = OFF_Q1 + TILE_BYTES;                     // PAIR: P0 | P1
    static constexpr int OFF_K = PAIR ? OFF_P + 2 * TILE_BYTES : OFF_Q1 + TILE_BYTES;
    static constexpr int OFF_V = PAIR ? OFF_K : OFF_K + KST * TILE_BYTES;
    static constexpr int OFF_BAR = PAIR ? OFF_K + KST * SLOT : OFF_V + 2 * TILE_BYTES;
    // + PAIR: s_free[2] (softmax holds S_g in registers), p_empty[2] (PV_g done: P_g reusable)
    static constexpr int NBAR = 14 + 2 * KST + 2 * (SDA_K2_PPARTS > 1 ? SDA_K2_PPARTS - 1 : 0) + (PAIR ? 4 : 0);
    static constexpr int OFF_SEG = OFF_BAR + NBAR * 8 + 16;
    static constexpr int OFF_XCH = OFF_SEG + (PAIR ? 8 : SEG_SLOTS) * 128;
    static constexpr int SMEM = OFF_XCH + (PAIR ? 0 : XCH_BYTES);
};
static_assert(Lay<true>::SMEM <= 232448, "pair form exceeds the 227 KB opt-in SMEM");
static_assert(Lay<false>::SMEM == SMEM, "layouts");
// 12 warps = 3 warpgroups so registers can move between them (setmaxnreg): softmax warps 0-7
// grow to 224, the TMA / MMA warpgroup (warps 8-9; 10-11 idle) shrinks to 56
#ifndef SDA_K2_SETMAXNREG
#define SDA_K2_SETMAXNREG 1
#endif
#if SDA_K2_SETMAXNREG
constexpr int THREADS = 384;
#else
constexpr int THREADS = 320;
#endif
constexpr int kSoftmaxRegs = 224, kIssueRegs = 56;
// split rows: 20 warps (primaries 0-7, issue warpgroup 8-11, helpers 12-19) launch at 96
// registers; setmaxnreg only moves registers within the CTA's own allocation, so
// 256 x 120 + 256 x 96 + 128 x 48 = 640 x 96
constexpr int kPrimRegs = 120, kHelpRegs = 96, kIssueRegsHelp = 48;
static_assert(256 * kPrimRegs + 256 * kHelpRegs + 128 * kIssueRegsHelp == 640 * 96, "register balance");
template <bool PAIR> struct Thr {
    static constexpr bool HELP = kHelp && !PAIR;
    static constexpr int N = HELP ? 640 : THREADS;
};
constexpr uint32_t COL_S0 = 0, COL_S1 = 128, COL_O0 = 256, COL_O1 = 384;
// Exponentials per 4 pairs computed on the FMA pipe (tc::exp2_fma2) instead of MUFU.EX2. Measured
// on C3 (exps batched ahead of the packing): 0 -> 489 us, 1 -> 485 us, 2 -> 547 us -- past one in
// four the added FMA-pipe instructions cost more issue time than the MUFU time they free.
#ifndef SDA_K2_EMU_OF4
#define SDA_K2_EMU_OF4 1
#endif
constexpr int kEmuOf4 = SDA_K2_EMU_OF4;
// Packed form (tc::exp2_fma2_packed: FADD2 / FFMA2, 5 issue slots per value against 8): the
// fraction of pairs on the FMA pipe in eighths (0 = the scalar form at kEmuOf4 of four). With the
// MMA warp's suspend-hint waits and additive descriptors, 1 of 8 packed is the best mix on C3:
// 439.7-440.7 us against 442.5-443.4 (scalar 1 of 4), 446.6-449.5 (all MUFU), 449.2-452.0 (2 of 8)
#ifndef SDA_K2_EMU_OF8P
#define SDA_K2_EMU_OF8P 1
#endif
constexpr int kEmuOf8P = SDA_K2_EMU_OF8P;
#ifndef SDA_K2_SUM_AFTER
#define SDA_K2_SUM_AFTER 1
#endif
#ifndef SDA_K2_SPEC
#define SDA_K2_SPEC 0
#endif
#ifndef SDA_K2_MAX4
#define SDA_K2_MAX4 0
#endif
static_assert(!kHelp || (SDA_K2_SETMAXNREG && !SDA_K2_SPEC), "split rows: setmaxnreg, no speculation");
}  // namespace k2tc

namespace k2tc {
// One unit of work = (request, q head, pair of 128-row Q tiles) over a range of 128-key tiles.
struct Seg {
    int64_t head_row;    // global Q row of the unit's first row
    int b;               // request
    int kvh;             // kv head (key set)
    int nrows;           // rows of the unit (<= 256)
    int len;             // keys of request b
    int t0, nkv;         // first unit-local key tile, tiles in this segment
    int split;           // split mode: output slot
    int unit, ub, nt;    // stream-K: unit index, its first tile in its group's linear order, its tiles
    bool two;            // second Q tile in use
    bool first;          // stream-K: the segment starts the CTA's range
};


__device__ __forceinline__ int len_of(const K2TcParams& p, int64_t b) {
    return p.kv_len ? p.kv_len[b] : (int)p.kv_cap;
}
__device__ __forceinline__ int ntile_of(const K2TcParams& p, int64_t b) { return (len_of(p, b) + TILE - 1) / TILE; }

// unit (request b, q head, Q-tile pair qp)
__device__ __forceinline__ void fill_unit(const K2TcParams& p, int b, int head, int qp, Seg& s) {
    s.b = b;
    s.kvh = head / (p.q_heads / p.kv_heads);
    s.head_row = ((int64_t)b * p.q_heads + head) * p.q_rows + (int64_t)qp * 2 * TILE;
    s.nrows = (int)min((int64_t)2 * TILE, p.q_rows - (int64_t)qp * 2 * TILE);
    s.two = s.nrows > TILE;
    s.len = len_of(p, b);
}

// split mode: the CTA's one segment -- blockIdx.z = request * n_splits + split;
//   normal : blockIdx.x = 256-row pair of Q tiles, blockIdx.y = q head
//   grouped: blockIdx.y = kv head; the tile rows are its G q heads x Lq rows
// split mode: segments per CTA (causal: the paired Q-tile pairs, 1 for the middle pair of an odd count)
__device__ __forceinline__ int split_nseg(const K2TcParams& p) {
    if (!p.causal) return 1;
    return (int)blockIdx.y == p.n_qpairs - 1 - (int)blockIdx.y ? 1 : 2;
}

__device__ __forceinline__ void split_seg(const K2TcParams& p, Seg& s, int idx = 0) {
    const int64_t b = blockIdx.z / p.n_splits;
    const int split = blockIdx.z % p.n_splits;
    const int G = p.q_heads / p.kv_heads;
    const int head = p.causal ? (int)blockIdx.x : (int)blockIdx.y;
    const int qp = p.causal ? (idx == 0 ? p.n_qpairs - 1 - (int)blockIdx.y : (int)blockIdx.y) : (int)blockIdx.x;
    s.b = (int)b;
    s.split = split;
    s.kvh = p.grouped ? head : head / G;
    s.head_row = p.grouped ? (b * p.q_heads + (int64_t)s.kvh * G) * p.q_rows
                           : (b * p.q_heads + head) * p.q_rows + (int64_t)qp * 2 * TILE;
    s.nrows = (int)(p.grouped ? (int64_t)G * p.q_rows : min((int64_t)2 * TILE, p.q_rows - (int64_t)qp * 2 * TILE));
    s.two = s.nrows > TILE;
    s.len = len_of(p, b);
    if (p.causal) {   // the pair's last row sees keys < its index + offset + 1: the tiles past are skipped
        const int64_t lim = (int64_t)qp * 2 * TILE + s.nrows + p.causal_offset;
        s.len = (int)max((int64_t)0, min((int64_t)s.len, lim));
    }
    // split ranges aligned to whole 128-key tiles
    const int ntile_all = (s.len + TILE - 1) / TILE;
    const int tps = (ntile_all + p.n_splits - 1) / p.n_splits;
    const int t0 = split * tps;
    const int t1 = min(ntile_all, t0 + tps);
    s.t0 = t0;
    s.nkv = t1 > t0 ? t1 - t0 : 0;
    s.unit = s.ub = s.nt = 0;
    s.first = true;
}

// Stream-K: the (request, q head) key tiles laid end to end = T tiles. The grid is NG groups of
// n_qpairs CTAs; CTA (group g, pair qp) takes the Q-tile pair qp of every (request, head) over
// tiles [T g / NG, T (g+1) / NG) -- so a group's CTAs walk the same keys in lockstep and read
// each K/V tile from HBM once (the L2 serves the others), as the split-mode grid does. A range
// covers the tail of one (request, head), whole ones, the head of another.
__device__ __forceinline__ int sk_lo(int T, int NG, int g) { return (int)((int64_t)T * g / NG); }

struct SkCursor {
    int lo, hi, pos, b, head, off, acc, nt;
};

__device__ __forceinline__ void sk_init(const K2TcParams& p, int T, int NG, int g, SkCursor& k) {
    k.lo = g < NG ? sk_lo(T, NG, g) : 0;
    k.hi = g < NG ? sk_lo(T, NG, g + 1) : 0;
    k.pos = k.lo;
    k.acc = k.b = k.nt = k.head = k.off = 0;
    if (k.pos >= k.hi) return;
    const int nhs = p.q_heads * (p.n_qpairs / p.sk_gq);   // (head, pair-subset) sequences per request
    for (;; ++k.b) {
        k.nt = ntile_of(p, k.b);
        if (k.pos < k.acc + nhs * k.nt) break;
        k.acc += nhs * k.nt;
    }
    k.head = (k.pos - k.acc) / k.nt;
    k.off = (k.pos - k.acc) % k.nt;
}

__device__ __forceinline__ bool sk_next(const K2TcParams& p, int qp, SkCursor& k, Seg& s) {
    if (k.pos >= k.hi) return false;
    const int nsub = p.n_qpairs / p.sk_gq, nhs = p.q_heads * nsub;
    const int head = k.head / nsub, qpair = (k.head % nsub) * p.sk_gq + qp;
    fill_unit(p, k.b, head, qpair, s);
    s.t0 = k.off;
    s.nkv = min(k.nt - k.off, k.hi - k.pos);
    s.split = 0;
    s.unit = (k.b * p.q_heads + head) * p.n_qpairs + qpair;
    s.ub = k.acc + k.head * k.nt;
    s.nt = k.nt;
    s.first = k.pos == k.lo;
    k.pos += s.nkv;
    k.off += s.nkv;
    if (k.off == k.nt) {
        k.off = 0;
        if (++k.head == nhs) {
            k.head = 0;
            k.acc += nhs * k.nt;
            ++k.b;
            while (k.pos < k.hi && (k.nt = ntile_of(p, k.b)) == 0) ++k.b;   // requests with no keys
        }
    }
    return true;
}

// A softmax warp's segment state waits out the tile loop in SMEM, so it holds no registers
// next to the 128 logits of a row (re-read through an opaque pointer).
struct SoftKeep {
    Seg seg;
    SkCursor cur;
    int T, NG;
};
static_assert(sizeof(SoftKeep) <= 128, "one 128-byte SMEM slot per softmax warp");
__device__ __forceinline__ SoftKeep* opaque(SoftKeep* k) {
    SoftKeep* r;
    asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(k));
    return r;
}

// group whose range holds linear tile x
__device__ __forceinline__ int sk_group_of(int x, int T, int NG) {
    int g = (int)min((int64_t)NG - 1, (int64_t)x * NG / T);
    while (g + 1 < NG && sk_lo(T, NG, g + 1) <= x) ++g;
    while (g > 0 && sk_lo(T, NG, g) > x) --g;
    return g;
}

// scratch slot (CTA, k): k = 0 the CTA's first segment, 1 its last, 2 whole units; O rows then stats
constexpr int64_t SK_SLOT = 2 * TILE * D + 2 * TILE * 2;
__device__ __forceinline__ float* sk_slot(const K2TcParams& p, int cta, int k) {
    return p.sk_buf + ((int64_t)cta * 3 + k) * SK_SLOT;
}

// 16 f32 of a thread's own output row (x inv) as two 256-bit stores: whole 32-byte sectors per
// lane instead of the half sectors of 16-byte stores (the thread-per-row epilogue)
__device__ __forceinline__ void store_row16(float* dst, const uint32_t (&o)[16], float inv) {
    if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 8 * h),
                         "f"(__uint_as_float(o[8 * h + 0]) * inv), "f"(__uint_as_float(o[8 * h + 1]) * inv),
                         "f"(__uint_as_float(o[8 * h + 2]) * inv), "f"(__uint_as_float(o[8 * h + 3]) * inv),
                         "f"(__uint_as_float(o[8 * h + 4]) * inv), "f"(__uint_as_float(o[8 * h + 5]) * inv),
                         "f"(__uint_as_float(o[8 * h + 6]) * inv), "f"(__uint_as_float(o[8 * h + 7]) * inv)
                         : "memory");
    } else {   // a caller's output view only 16-byte aligned
#pragma unroll
        for (int e = 0; e < 4; ++e)
            reinterpret_cast<float4*>(dst)[e] =
                make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                            __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
    }
}

__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
}  // namespace k2tc

template <bool PAIR>
__global__ void __launch_bounds__(k2tc::Thr<PAIR>::N, 1)
k2_prefill_tc_kernel(const K2TcParams p, const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                     const __grid_constant__ CUtensorMap vmap) {
    using namespace k2tc;
    using L = Lay<PAIR>;
    constexpr int KST = L::KST;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* const bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* const q_full = bars;
    uint64_t* const k_full = bars + 1;
    uint64_t* const k_empty = k_full + KST;
    uint64_t* const v_full = k_empty + KST;
    uint64_t* const v_empty = v_full + 2;
    uint64_t* const s_full = v_empty + 2;
    uint64_t* const p_full = s_full + 2;
    uint64_t* const o_final = p_full + 2;
    uint64_t* const q_empty = o_final + 2;
    uint64_t* const o_empty = q_empty + 1;
    // PSPLIT: part i (< kPParts - 1) of tile g's P is in TMEM -- one barrier per part, so each
    // completes once per tile (a barrier completing several phases ahead of its waiter would
    // leave the waiter's parity ambiguous)
    uint64_t* const p_part = o_empty + 2;
    uint64_t* const s_free = p_part + 2 * (kPParts > 1 ? kPParts - 1 : 0);   // PAIR only
    uint64_t* const p_empty = s_free + 2;                                     // PAIR only
    uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(bars + L::NBAR);
    // PAIR: rank 0 issues the MMAs and owns the barriers the pair's TMA bytes and softmax
    // arrivals complete on (both CTAs arrive there; commits multicast to both CTAs' copies)
    const uint32_t crank = PAIR ? tc::cluster_rank() : 0u;
    // softmax -> MMA hand-off. PAIR: one arrive per warp (its lanes ordered before it by
    // __syncwarp) on this CTA's barrier; rank 1's are forwarded to rank 0 by its relay warps
    auto arrive0 = [&](uint64_t* b) {
        if (PAIR) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) tc::mbar_arrive(b);
        } else {
            tc::mbar_arrive(b);
        }
    };
    auto commit = [&](uint64_t* b) {
        if (PAIR) tc::mma_commit_pair(b);
        else tc::mma_commit(b);
    };
    uint32_t* const sk_ticket = tmem_slot + 1;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // Work: split mode -- one segment per CTA: blockIdx.z = request * n_splits + split;
    //   normal : blockIdx.x = 256-row pair of Q tiles, blockIdx.y = q head
    //   grouped: blockIdx.y = kv head; the tile rows are its G q heads x Lq rows
    // stream-K mode (p.sk) -- a persistent CTA per SM walking its range of the linear tile order.
    int T_sk = 0, NG = 1;
    const int gq = p.sk ? p.sk_gq : 1;   // stream-K: CTAs per group
    const int grp = (int)blockIdx.x / gq, qp_sk = (int)blockIdx.x % gq;
    if (p.sk) {
        for (int64_t b = 0; b < p.n_batch; ++b) T_sk += ntile_of(p, b);
        T_sk *= p.q_heads * (p.n_qpairs / gq);
        // groups that take part in the range split: every range then holds >= 1 tile (ragged
        // kv_len can leave fewer tiles than groups; the other CTAs only serve empty requests)
        NG = max(1, min((int)gridDim.x / gq, T_sk));
    }
    // the CTA's segments, the same sequence in every warp role
    SkCursor cur;
    if (p.sk) sk_init(p, T_sk, NG, grp, cur);
    int lseg = 0;   // split mode: segments of this CTA taken so far
    auto next_seg = [&](Seg& sg) -> bool {
        if (p.sk) return sk_next(p, qp_sk, cur, sg);
        if (lseg >= split_nseg(p)) return false;
        split_seg(p, sg, lseg++);
        return true;
    };

    if (tid == 0) {
        tc::mbar_init(q_full, 1);
        tc::mbar_init(q_empty, PAIR ? 2 : 1);   // PAIR: released by both issuer warps
        for (int i = 0; i < KST; ++i) {
            tc::mbar_init(&k_full[i], 1);
            tc::mbar_init(&k_empty[i], PAIR ? 2 : 1);
        }
        // softmax arrivals per hand-off: a thread each; PAIR: a lane per warp, + rank 1's relay on rank 0
        const uint32_t NSOFT = PAIR ? (crank == 0 ? 5u : 4u) : 128u;
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&v_full[i], 1);
            tc::mbar_init(&v_empty[i], 1);
            tc::mbar_init(&s_full[i], 1);
            tc::mbar_init(&p_full[i], NSOFT);
            for (int part = 0; part + 1 < kPParts; ++part) tc::mbar_init(&p_part[i * (kPParts - 1) + part], NSOFT);
            tc::mbar_init(&o_final[i], 1);
            tc::mbar_init(&o_empty[i], NSOFT);
            if (PAIR) {
                tc::mbar_init(&s_free[i], NSOFT);
                tc::mbar_init(&p_empty[i], 1);
            }
        }
        tc::fence_mbar_init();
    }
    if (warp == 0) {
        if (PAIR) tc::tmem_alloc_pair<512>(tmem_slot);
        else tc::tmem_alloc<512>(tmem_slot);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (PAIR) tc::cluster_sync();   // both CTAs' barriers exist before any remote arrive / TMA byte
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    K2_CTA_STAMP(0);

    constexpr bool HX = Thr<PAIR>::HELP;
    if (warp >= 8 && (!HX || warp < 12)) {
#if SDA_K2_SETMAXNREG
      if constexpr (HX) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kIssueRegsHelp));
      else asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kIssueRegs));
#endif
      if (warp == 8) {
        // ------------------------------------------------------------------ TMA producer
        // K/V tiles run through the 2-stage rings continuously across segments (jj counts all
        // tiles of the CTA); a segment's Q is loaded after its first K/V tile is queued, once the
        // previous segment's MMAs have released the Q buffers
        if (lane == 0) {
            tc::prefetch_tmap(&qmap);
            tc::prefetch_tmap(&kmap);
            tc::prefetch_tmap(&vmap);
            int64_t jj = 0;
            int si = 0;
            Seg sg;
            auto load_q = [&](const Seg& s) {
                tc::mbar_arrive_expect_tx(q_full, (s.two ? 2 : 1) * TILE_BYTES);
                for (int g = 0; g < (s.two ? 2 : 1); ++g)
                    for (int kb = 0; kb < 2; ++kb)
                        tc::tma_load_2d(smem + (g ? OFF_Q1 : OFF_Q0) + kb * BLK, &qmap, kb * 64, (int)(s.head_row + g * TILE),
                                        q_full);
            };
            // PAIR: this CTA's Q tiles and K / V halves; rank 0's barriers count the pair's bytes
            auto load_q2 = [&](const Seg& s) {
                if (crank == 0) tc::mbar_arrive_expect_tx(q_full, 2 * (s.two ? 2 : 1) * TILE_BYTES);
                const uint32_t qf = tc::at_rank0(q_full);
                for (int g = 0; g < (s.two ? 2 : 1); ++g)
                    for (int kb = 0; kb < 2; ++kb)
                        tc::tma_load_2d_pair(smem + (g ? OFF_Q1 : OFF_Q0) + kb * BLK, &qmap, kb * 64, (int)(s.head_row + g * TILE), qf);
            };
            // ring item `it` into slot it % KST: a K half (keys 64 r .. 64 r + 63 of the tile, as two
            // [64 x 64] SW128 blocks) or a V half (d columns 64 r .. 64 r + 63 of its 128 keys)
            auto ring_load = [&](int64_t it, bool is_v, int64_t row0) {
                const int sl = (int)(it % KST);
                if (it >= KST) tc::mbar_wait(&k_empty[sl], (uint32_t)((it / KST - 1) & 1));
                if (crank == 0) tc::mbar_arrive_expect_tx(&k_full[sl], 2 * L::SLOT);
                const uint32_t fb = tc::at_rank0(&k_full[sl]);
                uint8_t* const dst = smem + L::OFF_K + sl * L::SLOT;
                if (is_v) {
                    tc::tma_load_2d_pair(dst, &vmap, 64 * (int)crank, (int)row0, fb);
                } else {
                    for (int kb = 0; kb < 2; ++kb)
                        tc::tma_load_2d_pair(dst + kb * (L::SLOT / 2), &kmap, kb * 64, (int)(row0 + 64 * crank), fb);
                }
            };
            while (PAIR && next_seg(sg)) {
                if (sg.nkv == 0) continue;
                if (si == 0) load_q2(sg);
                const int64_t kvrow0 = (((int64_t)sg.b * p.kv_heads + sg.kvh) * p.kv_cap) + (int64_t)sg.t0 * TILE;
                ring_load(jj++, false, kvrow0);                       // K(0)
                if (si > 0) {
                    tc::mbar_wait(q_empty, (uint32_t)((si - 1) & 1));
                    load_q2(sg);
                }
                if (sg.nkv > 1) ring_load(jj++, false, kvrow0 + TILE);   // K(1)
                for (int64_t j = 0; j < sg.nkv; ++j) {
                    ring_load(jj++, true, kvrow0 + j * TILE);                              // V(j)
                    if (j + 2 < sg.nkv) ring_load(jj++, false, kvrow0 + (j + 2) * TILE);   // K(j+2)
                }
                ++si;
            }
            while (!PAIR && next_seg(sg)) {
                if (sg.nkv == 0) continue;
                if (si == 0) load_q(sg);   // the first segment's Q ahead of its K/V (nothing to wait for)
                const int64_t kvrow0 = (((int64_t)sg.b * p.kv_heads + sg.kvh) * p.kv_cap) + (int64_t)sg.t0 * TILE;
                for (int64_t j = 0; j < sg.nkv; ++j, ++jj) {
                    const int st = (int)(jj & 1);
                    const uint32_t ph = (uint32_t)(((jj >> 1) - 1) & 1);
                    const int sk = (int)(jj % KST);
                    if (jj >= KST) tc::mbar_wait(&k_empty[sk], (uint32_t)((jj / KST - 1) & 1));
                    tc::mbar_arrive_expect_tx(&k_full[sk], TILE_BYTES);
                    for (int kb = 0; kb < 2; ++kb)
                        tc::tma_load_2d(smem + L::OFF_K + sk * TILE_BYTES + kb * BLK, &kmap, kb * 64, (int)(kvrow0 + j * TILE), &k_full[sk]);
                    if (jj >= 2) tc::mbar_wait(&v_empty[st], ph);
                    tc::mbar_arrive_expect_tx(&v_full[st], TILE_BYTES);
                    for (int kb = 0; kb < 2; ++kb)
                        tc::tma_load_2d(smem + L::OFF_V + st * TILE_BYTES + kb * BLK, &vmap, kb * 64, (int)(kvrow0 + j * TILE), &v_full[st]);
                    if (j == 0 && si > 0) {   // later segments: once the previous one's MMAs release Q
                        tc::mbar_wait(q_empty, (uint32_t)((si - 1) & 1));
                        load_q(sg);
                    }
                }
                ++si;
            }
        }
      } else if (warp == 9 || (PAIR && crank == 0 && warp == 10)) {
        // ------------------------------------------------------------------ MMA issuer
        // (PAIR: warp 9 issues Q tile 0's MMAs, warp 10 tile 1's -- two issuers, so neither
        // tile's MMAs queue behind the other tile's P)
        // the whole warp runs the loop (warp-uniform descriptors); the elected lane issues
        const bool leader = tc::elect_one();
        constexpr uint32_t IDESC_S = tc::idesc_bf16_f32(128, 128, false, false);   // Q K^T, both K-major
        constexpr uint32_t IDESC_O = tc::idesc_bf16_f32(128, 128, false, true);    // P V, V MN-major
        const uint32_t q0 = tc::smem_u32(smem + OFF_Q0), q1 = tc::smem_u32(smem + OFF_Q1);
        const uint32_t kbase = tc::smem_u32(smem + L::OFF_K), vbase = tc::smem_u32(smem + L::OFF_V);
        const uint32_t pbase = tc::smem_u32(smem + L::OFF_P);   // PAIR
        auto issue_s = [&](int g, int st) {
            const uint32_t qa = g ? q1 : q0;
            const uint32_t kb = kbase + st * TILE_BYTES;
            const uint32_t d_tmem = tmem + (g ? COL_S1 : COL_S0);
            // descriptors as base + (byte offset >> 4): the start-address field is the low 14 bits
            // and SMEM offsets stay below 256 KB, so the add never carries out of it -- one uniform
            // add per operand instead of the shift / mask / or of a fresh descriptor (the MMA warp
            // shares SMSP 1's issue slots with two softmax warps)
            const uint64_t da0 = tc::sw128_desc(qa, 16, 1024), db0 = tc::sw128_desc(kb, 16, 1024);
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
                const uint32_t off = ((k >> 2) * BLK + (k & 3) * 32) >> 4;
                if (leader) tc::mma_bf16_ss(d_tmem, da0 + off, db0 + off, IDESC_S, k > 0 ? 1u : 0u);
            }
            if (leader) tc::mma_commit(&s_full[g]);
        };
        auto issue_pv = [&](int g, int st, bool acc, int k0, int k1) {
            const uint32_t vb = vbase + st * TILE_BYTES;
            const uint32_t d_tmem = tmem + (g ? COL_O1 : COL_O0);
            const uint32_t p_tmem = tmem + (g ? COL_S1 : COL_S0);
            const uint64_t db0 = tc::sw128_desc(vb, BLK, 1024);
#pragma unroll
            for (int k = k0; k < k1; ++k) {   // 16 keys per step: P columns 8k.., V rows 16k..
                if (leader) tc::mma_bf16_ts(d_tmem, p_tmem + k * 8, db0 + (uint32_t)(k * 2048 >> 4), IDESC_O, (acc || k > 0) ? 1u : 0u);
            }
        };
        // PV of tile g: with PSPLIT the first 64 keys go as soon as their P is in TMEM
        auto pv = [&](int g, int st, bool acc, uint32_t n) {   // n: P tiles of Q tile g so far
            const uint32_t ph = n & 1;
#if SDA_K2_PSPLIT
            constexpr int KPP = TILE / 16 / kPParts;   // PV k-steps per part
#pragma unroll
            for (int part = 0; part + 1 < kPParts; ++part) {   // one barrier per part
                K2_WAIT_P(&p_part[g * (kPParts - 1) + part], ph);
                tc::tc_fence_after();
                issue_pv(g, st, acc, part * KPP, (part + 1) * KPP);
            }
            K2_WAIT_P(&p_full[g], ph);
            tc::tc_fence_after();
            issue_pv(g, st, true, (kPParts - 1) * KPP, TILE / 16);
#else
            K2_WAIT_P(&p_full[g], ph);
            tc::tc_fence_after();
            issue_pv(g, st, acc, 0, TILE / 16);
#endif
        };
        int64_t jj = 0;
        int si = 0;
        uint32_t pc[2] = {0u, 0u}, ou[2] = {0u, 0u};   // P tiles consumed / segments accumulated, per Q tile
        Seg sg;
        // ---- PAIR (rank 0 only): M = 256 MMAs over both CTAs' rows, one issuer warp per Q tile g.
        // S runs two tiles ahead of P: per step PV_g(j) then S_g(j+2) -- PV_g(j) once P_g(j) is in
        // both CTAs' SMEM, S_g(j+2) once both CTAs' softmax hold S_g(j+1) in registers (s_free).
        // Ring slots and Q are released by both issuers (k_empty / q_empty count 2).
        const int gi = warp - 9;
        constexpr uint32_t IDESC_S2 = tc::idesc_bf16_f32(256, 128, false, false);
        constexpr uint32_t IDESC_O2 = tc::idesc_bf16_f32(256, 128, false, true);
        uint32_t ns[2] = {0u, 0u};   // S tiles issued per Q tile
        auto s_next2 = [&](int g, int sl) {
            if (ns[g] > 0) tc::mbar_wait_cluster(&s_free[g], (ns[g] - 1) & 1);
            tc::tc_fence_after();
            const uint32_t qa = g ? q1 : q0;
            const uint32_t kb = kbase + sl * L::SLOT;
            const uint64_t da0 = tc::sw128_desc(qa, 16, 1024), db0 = tc::sw128_desc(kb, 16, 1024);   // (as issue_s)
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
                const uint64_t da = da0 + (uint32_t)(((k >> 2) * BLK + (k & 3) * 32) >> 4);
                const uint64_t db = db0 + (uint32_t)(((k >> 2) * (L::SLOT / 2) + (k & 3) * 32) >> 4);
                if (leader) tc::mma_bf16_ss_pair(tmem + (g ? COL_S1 : COL_S0), da, db, IDESC_S2, k > 0 ? 1u : 0u);
            }
            if (leader) tc::mma_commit_pair(&s_full[g]);
            ++ns[g];
        };
        auto pv2 = [&](int g, int sl, bool acc, uint32_t n) {
            const uint32_t ph = n & 1;
            const uint32_t vb = kbase + sl * L::SLOT;
            const uint32_t pa = pbase + g * TILE_BYTES;
            const uint64_t dp0 = tc::sw128_desc(pa, 16, 1024), dv0 = tc::sw128_desc(vb, BLK, 1024);
            auto issue = [&](int k0, int k1, bool a) {
#pragma unroll
                for (int k = k0; k < k1; ++k) {
                    const uint64_t da = dp0 + (uint32_t)(((k >> 2) * BLK + (k & 3) * 32) >> 4);
                    const uint64_t db = dv0 + (uint32_t)(k * 2048 >> 4);
                    if (leader) tc::mma_bf16_ss_pair(tmem + (g ? COL_O1 : COL_O0), da, db, IDESC_O2, (a || k > 0) ? 1u : 0u);
                }
            };
            constexpr int KPP = TILE / 16 / kPParts;
#pragma unroll
            for (int part = 0; part + 1 < kPParts; ++part) {
                tc::mbar_wait_cluster(&p_part[g * (kPParts - 1) + part], ph);
                tc::tc_fence_after();
                issue(part * KPP, (part + 1) * KPP, acc);
            }
            if (g == 0) K2_STAMP(18, n);
            tc::mbar_wait_cluster(&p_full[g], ph);
            if (g == 0) K2_STAMP(19, n);
            tc::tc_fence_after();
            issue((kPParts - 1) * KPP, TILE / 16, kPParts > 1 ? true : acc);
        };
        while (PAIR && crank == 0 && next_seg(sg)) {
            if (sg.nkv == 0) continue;
            tc::mbar_wait_cluster(q_full, (uint32_t)(si & 1));
            for (int t = 0; t < 2 && t < sg.nkv; ++t) {   // K(0), K(1): S_g(0), S_g(1)
                const int sl = (int)(jj % KST);
                tc::mbar_wait_cluster(&k_full[sl], (uint32_t)((jj / KST) & 1));
                s_next2(gi, sl);
                if (leader) tc::mma_commit_pair(&k_empty[sl]);
                ++jj;
            }
            for (int64_t j = 0; j < sg.nkv; ++j) {
                const int slv = (int)(jj % KST);   // V(j)
                const int64_t jk = jj + 1;         // K(j+2), if any
                const int slk = (int)(jk % KST);
                const bool more = j + 2 < sg.nkv;
                if (gi == 0) K2_STAMP(6, j);
                tc::mbar_wait_cluster(&k_full[slv], (uint32_t)((jj / KST) & 1));
                if (gi == 0) K2_STAMP(7, j);
                if (j == 0 && ou[gi] > 0) tc::mbar_wait_cluster(&o_empty[gi], (ou[gi] - 1) & 1);
                K2_STAMP(4 + gi, j);
                pv2(gi, slv, j > 0, pc[gi]);
                ++pc[gi];
                if (leader) tc::mma_commit_pair(&p_empty[gi]);
                if (j + 1 == sg.nkv && leader) tc::mma_commit_pair(&o_final[gi]);
                if (more) {
                    if (gi == 0) K2_STAMP(9, j);
                    tc::mbar_wait_cluster(&k_full[slk], (uint32_t)((jk / KST) & 1));
                    if (gi == 0) K2_STAMP(10, j);
                    s_next2(gi, slk);
                }
                if (leader) tc::mma_commit_pair(&k_empty[slv]);
                ++jj;
                if (more) {
                    if (leader) tc::mma_commit_pair(&k_empty[slk]);
                    ++jj;
                }
            }
            ++ou[gi];
            if (leader) tc::mma_commit_pair(q_empty);
            ++si;
        }
        while (!PAIR && next_seg(sg)) {
            if (sg.nkv == 0) continue;
            const bool two = sg.two;
            tc::mbar_wait(q_full, (uint32_t)(si & 1));
            tc::mbar_wait(&k_full[jj % KST], (uint32_t)((jj / KST) & 1));
            tc::tc_fence_after();
            issue_s(0, (int)(jj % KST));
            if (two) issue_s(1, (int)(jj % KST));
            if (leader) tc::mma_commit(&k_empty[jj % KST]);
            for (int64_t j = 0; j < sg.nkv; ++j) {
                const int64_t J = jj + j;
                const int st = (int)(J & 1);
                const uint32_t ph = (uint32_t)((J >> 1) & 1);
                K2_STAMP(6, J);
                tc::mbar_wait(&v_full[st], ph);
                K2_STAMP(7, J);
                // O0 is reused from the previous segment once its epilogue has read it
                if (j == 0 && ou[0] > 0) tc::mbar_wait(&o_empty[0], (ou[0] - 1) & 1);
                K2_STAMP(4, J);
                pv(0, st, j > 0, pc[0]);
                ++pc[0];
                if (!two && leader) tc::mma_commit(&v_empty[st]);
                if (j + 1 == sg.nkv && leader) tc::mma_commit(&o_final[0]);
                const int sn = (int)((J + 1) % KST);
                if (j + 1 < sg.nkv) {
                    K2_STAMP(9, J);
                    tc::mbar_wait(&k_full[sn], (uint32_t)(((J + 1) / KST) & 1));
                    K2_STAMP(10, J);
                    tc::tc_fence_after();
                    issue_s(0, sn);
                    if (!two && leader) tc::mma_commit(&k_empty[sn]);
                }
                if (!two) continue;
                K2_STAMP(8, J);
                if (j == 0 && ou[1] > 0) tc::mbar_wait(&o_empty[1], (ou[1] - 1) & 1);
                K2_STAMP(5, J);
                pv(1, st, j > 0, pc[1]);
                ++pc[1];
                if (leader) tc::mma_commit(&v_empty[st]);
                if (j + 1 == sg.nkv && leader) tc::mma_commit(&o_final[1]);
                if (j + 1 < sg.nkv) {
                    issue_s(1, sn);
                    if (leader) tc::mma_commit(&k_empty[sn]);
                }
            }
            ++ou[0];
            if (two) ++ou[1];
            if (leader) tc::mma_commit(q_empty);   // Q buffers free once this segment's MMAs are done
            jj += sg.nkv;
            ++si;
        }
      } else if (PAIR && crank == 1 && lane == 0) {
        // ------------------------------------------------------------------ relay (PAIR, rank 1)
        // Rank 1's softmax warps arrive on their own CTA's copies of s_free / p_part / p_full /
        // o_empty (cta scope); warp 10 (Q tile 0) / 11 (tile 1) forwards each completed phase to
        // rank 0's barrier with one relaxed cluster arrive. (A release.cluster arrive costs a
        // MEMBAR.GPU, ~0.7 us: per softmax warp and hand-off that was ~1 us of every tile, and
        // still ~0.7 us of hand-off latency in the relay.)
        const int g = warp - 10;
        uint32_t n_t = 0, n_o = 0;   // tiles / segments relayed
        Seg sg;
        while (next_seg(sg)) {
            if (!(g == 0 || sg.two)) continue;
            for (int j = 0; j < sg.nkv; ++j, ++n_t) {
                K2_WAIT_RELAY(&s_free[g], n_t & 1);
                tc::mbar_arrive_remote_relaxed(tc::at_rank0(&s_free[g]));
                for (int part = 0; part + 1 < kPParts; ++part) {
                    K2_WAIT_RELAY(&p_part[g * (kPParts - 1) + part], n_t & 1);
                    tc::mbar_arrive_remote_relaxed(tc::at_rank0(&p_part[g * (kPParts - 1) + part]));
                }
                K2_WAIT_RELAY(&p_full[g], n_t & 1);
                if (g == 0) K2_STAMP1(20, n_t);
                tc::mbar_arrive_remote_relaxed(tc::at_rank0(&p_full[g]));
            }
            if (p.sk || sg.nkv > 0) {
                K2_WAIT_RELAY(&o_empty[g], n_o & 1);
                tc::mbar_arrive_remote_relaxed(tc::at_rank0(&o_empty[g]));
                ++n_o;
            }
        }
      }
    } else if (HX && warp >= 12) {
        // (helpers stay at the launch's 96 registers)
        // ------------------------------------------------------------------ split-row helpers
        // keys 64-127 of every tile for the rows of primary warp (warp - 12): the same segment
        // sequence, S loads, max exchange, base updates and row sum as the primary's half; no O
        // rescale (the primary rescales all of O_g before it hands over P's first half, and PV
        // waits for both halves) and no epilogue
        const int hw = warp - 12;
        const int g = hw >> 2;
        const int row = (hw & 3) * 32 + lane;
        const uint32_t s_col = tmem + (g ? COL_S1 : COL_S0) + ((uint32_t)((hw & 3) * 32) << 16);
        float* const xch = reinterpret_cast<float*>(smem + L::OFF_XCH);
        const uint32_t bar_id = 2u + (uint32_t)(g * 4 + (hw & 3));
        SoftKeep* const keep = reinterpret_cast<SoftKeep*>(smem + L::OFF_SEG) + 8 + hw;
        if (lane == 0) keep->cur = cur;
        __syncwarp();
        uint32_t sc = 0, segc = 0;
        Seg sg0;
        for (;;) {
            if (!p.sk) {
                if (lseg >= split_nseg(p)) break;
                split_seg(p, sg0, lseg++);
            } else {
                SoftKeep* const k = opaque(keep);
                SkCursor c = k->cur;
                const bool ok = sk_next(p, (int)blockIdx.x % p.sk_gq, c, sg0);
                __syncwarp();
                if (lane == 0) k->cur = c;
                __syncwarp();
                if (!ok) break;
            }
            const int nkv = sg0.nkv;
            const bool group_live = g == 0 || sg0.two;
            const bool warp_live = g * TILE + (hw & 3) * 32 < sg0.nrows;
            int kv_left = sg0.len - sg0.t0 * TILE;
            if (p.causal) {
                const int64_t qrow = sg0.head_row % p.q_rows + (int64_t)g * TILE + row;
                const int64_t lim = min((int64_t)len_of(p, sg0.b), qrow + p.causal_offset + 1);
                kv_left = (int)max((int64_t)-TILE, lim - (int64_t)sg0.t0 * TILE);
            }
            float m_run = -INFINITY, m_use = -INFINITY, l = 0.f;
            for (int j = 0; group_live && j < nkv; ++j) {
                K2_WAIT_S(&s_full[g], sc & 1);
                const uint32_t par = sc & 1;
                ++sc;
                tc::tc_fence_after();
                if ((hw & 3) == 0 && lane == 0) K2_STAMP(g ? 22 : 18, j);
                if (!warp_live) {
                    tc::tc_fence_before();
                    tc::mbar_arrive(&p_full[g]);
                    continue;
                }
                uint32_t s[64];
#pragma unroll
                for (int c = 0; c < 4; ++c) tc::tmem_ld16(s_col + 64 + c * 16, s + c * 16);
                tc::tmem_ld_wait();
                const int valid = kv_left - j * TILE - 64;
                if (valid < 64) {
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        if (i >= valid) s[i] = 0xFF800000u;
                }
                float mr0 = -INFINITY, mr1 = -INFINITY;
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    mr0 = tc::fmax3(mr0, __uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
                    mr1 = tc::fmax3(mr1, __uint_as_float(s[2 * i + 2]), __uint_as_float(s[2 * i + 3]));
                }
                float mt = fmaxf(mr0, mr1) * p.scale_log2;
                xch[(par * 2 + 1) * 256 + g * 128 + row] = mt;
                asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
                mt = fmaxf(mt, xch[(par * 2 + 0) * 256 + g * 128 + row]);
                const float m_new = fmaxf(m_run, mt);
                m_run = m_new;
                if (m_new > m_use + 8.f) {
                    if (m_use > -INFINITY) l *= ex2(m_use - m_new);
                    m_use = m_new;
                }
                const float mu = (m_use == -INFINITY) ? 0.f : m_use;
                const uint64_t sc2 = tc::f2(p.scale_log2, p.scale_log2), nmu2 = tc::f2(-mu, -mu);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    float x0, x1, p0, p1;
                    tc::f2_split(tc::ffma2(tc::f2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, nmu2), x0, x1);
                    if (kEmuOf8P > 0 && (i & 7) < kEmuOf8P) {
                        tc::exp2_fma2_packed(x0, x1, p0, p1);
                    } else if (kEmuOf8P == 0 && (i & 3) < kEmuOf4) {
                        tc::exp2_fma2(x0, x1, p0, p1);
                    } else {
                        p0 = ex2(x0);
                        p1 = ex2(x1);
                    }
                    s[2 * i] = __float_as_uint(p0);
                    s[2 * i + 1] = __float_as_uint(p1);
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        pk[e] = tc::pack_bf16(__uint_as_float(s[16 * c + 2 * e]), __uint_as_float(s[16 * c + 2 * e + 1]));
                    tc::tmem_st8(s_col + 32 + c * 8, pk);
                }
                tc::tmem_st_wait();
                tc::tc_fence_before();
                if ((hw & 3) == 0 && lane == 0) K2_STAMP(g ? 23 : 19, j);
                tc::mbar_arrive(&p_full[g]);
                uint64_t acc[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) acc[a] = tc::f2(0.f, 0.f);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    acc[i & 3] = tc::fadd2(acc[i & 3], tc::f2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])));
                float a0, a1, b0, b1, c0, c1, d0, d1;
                tc::f2_split(acc[0], a0, a1);
                tc::f2_split(acc[1], b0, b1);
                tc::f2_split(acc[2], c0, c1);
                tc::f2_split(acc[3], d0, d1);
                l += ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
            }
            if (group_live) {   // this half's row sum to the primary (double-buffered by segment)
                xch[2 * 2 * 2 * 128 + (segc & 1) * 256 + g * 128 + row] = l;
                asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
            }
            ++segc;
        }
    } else {
#if SDA_K2_SETMAXNREG
        if constexpr (HX) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kPrimRegs));
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftmaxRegs));
#endif
        // ------------------------------------------------------------------ softmax groups
        const int g = warp >> 2;                               // Q tile
        const int row = (warp & 3) * 32 + lane;                // TMEM lane = tile row
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t s_col = tmem + (g ? COL_S1 : COL_S0) + lane_off;
        const uint32_t o_col = tmem + (g ? COL_O1 : COL_O0) + lane_off;
        uint32_t sc = 0, oc = 0;                               // S tiles / segments seen by this group
        SoftKeep* const keep = reinterpret_cast<SoftKeep*>(smem + L::OFF_SEG) + warp;
        // split rows: this warp's half of the exchange with helper warp 12 + warp
        float* const xch = reinterpret_cast<float*>(smem + L::OFF_XCH);
        const uint32_t bar_id = 2u + (uint32_t)warp;
        uint32_t segc = 0;
        constexpr int NV = HX ? 64 : 128;   // logits of a row this thread takes per tile
        static_assert(!PAIR || (SDA_K2_SUM_AFTER && !SDA_K2_SPEC), "pair form: row sum after P, no speculation");
        // PAIR: this row of P_g in SMEM (SW128 K-major: 64-key blocks of 128-byte rows, 16-byte
        // chunks XOR-swizzled by row & 7 -- 8 consecutive rows cover all banks)
        const uint32_t p_row = tc::smem_u32(smem + L::OFF_P + g * TILE_BYTES) + (uint32_t)row * 128u;
        if (lane == 0) {
            keep->cur = cur;
            keep->T = T_sk;
            keep->NG = NG;
        }
        __syncwarp();
        auto soft_next = [&](Seg& sg) -> bool {
            if (!p.sk) {
                if (lseg >= split_nseg(p)) return false;
                split_seg(p, sg, lseg++);
                return true;
            }
            SoftKeep* const k = opaque(keep);
            SkCursor c = k->cur;
            const bool ok = sk_next(p, (int)blockIdx.x % p.sk_gq, c, sg);
            __syncwarp();
            if (lane == 0) k->cur = c;
            __syncwarp();
            return ok;
        };
        Seg sg0;
        int si_tr = 0;   // segment index (trace builds only)
        (void)si_tr;
        while (soft_next(sg0)) {
            if (tid == 0) K2_STAMP(11, si_tr);
            const int nkv = sg0.nkv;
            const bool group_live = g == 0 || sg0.two;
            // warps whose 32 rows are all past the unit's rows only keep the barrier protocol going
            const bool warp_live = g * TILE + (warp & 3) * 32 < sg0.nrows;
            int kv_left = sg0.len - sg0.t0 * TILE;                   // keys from the segment's first tile
            if (p.causal) {   // this thread's row: keys <= its span index + offset (and < kv_len)
                const int64_t qrow = sg0.head_row % p.q_rows + (int64_t)g * TILE + row;
                const int64_t lim = min((int64_t)len_of(p, sg0.b), qrow + p.causal_offset + 1);
                kv_left = (int)max((int64_t)-TILE, lim - (int64_t)sg0.t0 * TILE);
            }
            if (lane == 0) keep->seg = sg0;
            __syncwarp();
            float m_run = -INFINITY, m_use = -INFINITY, l = 0.f;
            for (int j = 0; group_live && j < nkv; ++j) {
                K2_WAIT_S(&s_full[g], sc & 1);
                ++sc;
                tc::tc_fence_after();
                if ((warp & 3) == 0 && lane == 0) K2_STAMP(g, j);
                // PAIR: P_g(t) may go into SMEM once PV_g(t-1) is done (t = sc - 1, this group's tiles)
                bool pe_pending = PAIR && sc >= 2;
                auto wait_pe = [&]() {
                    if (pe_pending) {
                        if (warp == 0 && lane == 0) K2_STAMP(16, j);
                        tc::mbar_wait(&p_empty[g], (sc - 2) & 1);
                        if (warp == 0 && lane == 0) K2_STAMP(17, j);
                        tc::tc_fence_after();
                        pe_pending = false;
                    }
                };
                if (!warp_live) {
                    tc::tc_fence_before();
                    if (PAIR) {
                        // its P arrivals wait for PV_g(t-1) like the live warps' do: S_g(t) can be
                        // in before the live warps have announced P_g(t-1), and an early arrival
                        // would complete that phase of p_full
                        arrive0(&s_free[g]);
                        wait_pe();
                    }
#if SDA_K2_PSPLIT
                    for (int part = 0; part + 1 < kPParts; ++part) arrive0(&p_part[g * (kPParts - 1) + part]);
#endif
                    if (!HX) arrive0(&p_full[g]);   // (split rows: the helper completes p_full)
                    continue;
                }
                uint32_t s[128];
                const int valid = kv_left - (int)j * TILE;            // keys of this tile still in range
                auto load_s = [&]() {
#pragma unroll
                    for (int c = 0; c < NV / 16; ++c) tc::tmem_ld16(s_col + c * 16, s + c * 16);
                    tc::tmem_ld_wait();
                    if (valid < NV) {                                 // only the unit's last tile
#pragma unroll
                        for (int i = 0; i < NV; ++i)
                            if (i >= valid) s[i] = 0xFF800000u;       // -inf
                    }
                };
                // p = exp2(s * scale - mu) in place (one packed FFMA2 per two logits), all 128 first:
                // the MUFU ops issue back to back instead of each waiting on its consumer. With
                // `with_max` the row max of the raw logits is taken in the same pass.
                auto exp_range = [&](float mu, bool with_max, float& mr0, float& mr1, int i0, int i1) {
                    const uint64_t sc2 = tc::f2(p.scale_log2, p.scale_log2), nmu2 = tc::f2(-mu, -mu);
#pragma unroll
                    for (int i = i0; i < i1; ++i) {
                        const float r0 = __uint_as_float(s[2 * i]), r1 = __uint_as_float(s[2 * i + 1]);
                        if (with_max) {
                            if (i & 1) mr1 = tc::fmax3(mr1, r0, r1);
                            else mr0 = tc::fmax3(mr0, r0, r1);
                        }
                        float x0, x1;
                        tc::f2_split(tc::ffma2(tc::f2(r0, r1), sc2, nmu2), x0, x1);
                        float p0, p1;
                        if (kEmuOf8P > 0 && (i & 7) < kEmuOf8P) {
                            tc::exp2_fma2_packed(x0, x1, p0, p1);
                        } else if (kEmuOf8P == 0 && (i & 3) < kEmuOf4) {
                            tc::exp2_fma2(x0, x1, p0, p1);
                        } else {
                            p0 = ex2(x0);
                            p1 = ex2(x1);
                        }
                        s[2 * i] = __float_as_uint(p0);
                        s[2 * i + 1] = __float_as_uint(p1);
                    }
                };
                auto exp_pass = [&](float mu, bool with_max, float& mr0, float& mr1) { exp_range(mu, with_max, mr0, mr1, 0, 64); };
                load_s();
                if (PAIR) {   // S_g is in registers: the MMA may compute S_g(j+1) into the same columns
                    tc::tc_fence_before();
                    arrive0(&s_free[g]);
                }
                // PAIR: keys 8cc .. 8cc+7 of this row of P into SMEM
                auto st_chunk = [&](int cc) {
                    const uint32_t a = p_row + (uint32_t)(cc >> 3) * BLK + ((uint32_t)((cc & 7) ^ (row & 7)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                                 "r"(tc::pack_bf16(__uint_as_float(s[8 * cc + 0]), __uint_as_float(s[8 * cc + 1]))),
                                 "r"(tc::pack_bf16(__uint_as_float(s[8 * cc + 2]), __uint_as_float(s[8 * cc + 3]))),
                                 "r"(tc::pack_bf16(__uint_as_float(s[8 * cc + 4]), __uint_as_float(s[8 * cc + 5]))),
                                 "r"(tc::pack_bf16(__uint_as_float(s[8 * cc + 6]), __uint_as_float(s[8 * cc + 7])))
                                 : "memory");
                };
                float mr0 = -INFINITY, mr1 = -INFINITY;
#if SDA_K2_SPEC
                // speculative: once every row of the warp has a base, exponentiate against it with
                // the tile max in the same pass (the max no longer sits between the S load and the
                // exponentials); a row whose max grew by more than 8 re-reads S from TMEM below
                const bool spec = __all_sync(0xffffffffu, m_use > -INFINITY);
#else
                constexpr bool spec = false;
#endif
                if (spec) {
                    exp_pass(m_use, true, mr0, mr1);
                } else {
                    // row max on the raw logits (scale > 0), two new values per 3-input max
#if SDA_K2_MAX4
                    // four independent chains: half the dependent FMNMX3 latency of two
                    float mr2 = -INFINITY, mr3 = -INFINITY;
#pragma unroll
                    for (int i = 0; i < 64; i += 4) {
                        mr0 = tc::fmax3(mr0, __uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
                        mr1 = tc::fmax3(mr1, __uint_as_float(s[2 * i + 2]), __uint_as_float(s[2 * i + 3]));
                        mr2 = tc::fmax3(mr2, __uint_as_float(s[2 * i + 4]), __uint_as_float(s[2 * i + 5]));
                        mr3 = tc::fmax3(mr3, __uint_as_float(s[2 * i + 6]), __uint_as_float(s[2 * i + 7]));
                    }
                    mr0 = fmaxf(mr0, mr2);
                    mr1 = fmaxf(mr1, mr3);
#else
#pragma unroll
                    for (int i = 0; i < NV / 2; i += 2) {
                        mr0 = tc::fmax3(mr0, __uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
                        mr1 = tc::fmax3(mr1, __uint_as_float(s[2 * i + 2]), __uint_as_float(s[2 * i + 3]));
                    }
#endif
                }
                float mt = fmaxf(mr0, mr1) * p.scale_log2;
                if (HX) {   // the row's other half: the helper's tile max
                    const uint32_t par = (sc - 1) & 1;
                    xch[(par * 2 + 0) * 256 + g * 128 + row] = mt;
                    asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
                    mt = fmaxf(mt, xch[(par * 2 + 1) * 256 + g * 128 + row]);
                    if (warp == 0 && lane == 0) K2_STAMP(20, j);
                }
                const float m_new = fmaxf(m_run, mt);
                m_run = m_new;
                // lazy rescale: keep the exponent base unless the max grew by more than 8 (x256)
                const bool need = m_new > m_use + 8.f;
                if (__any_sync(0xffffffffu, need && j > 0 && m_use > -INFINITY)) {
                    wait_pe();   // PAIR: O_g holds PV_g(j-1) only once it has completed
                    const float alpha = (need && m_use > -INFINITY) ? ex2(m_use - m_new) : 1.f;
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        uint32_t o[8];
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                     : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]),
                                       "=r"(o[7])
                                     : "r"(o_col + c * 8));
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 8; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                        tc::tmem_st8(o_col + c * 8, o);
                    }
                    tc::tmem_st_wait();
                }
                if (need) {
                    if (m_use > -INFINITY) l *= ex2(m_use - m_new);
                    m_use = m_new;
                }
                if (HX) {
                    // keys 0-63: P into TMEM columns 0-31, announced on p_part; the helper
                    // announces keys 64-127 on p_full
                    exp_range((m_use == -INFINITY) ? 0.f : m_use, false, mr0, mr1, 0, 32);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t pk[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            pk[e] = tc::pack_bf16(__uint_as_float(s[16 * c + 2 * e]), __uint_as_float(s[16 * c + 2 * e + 1]));
                        tc::tmem_st8(s_col + c * 8, pk);
                    }
                    tc::tmem_st_wait();
                    tc::tc_fence_before();
                    if ((warp & 3) == 0 && lane == 0) K2_STAMP(2 + g, j);
                    arrive0(&p_part[g * (kPParts - 1)]);
                    uint64_t acc[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) acc[a] = tc::f2(0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        acc[i & 3] = tc::fadd2(acc[i & 3], tc::f2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])));
                    float a0, a1, b0, b1, c0, c1, d0, d1;
                    tc::f2_split(acc[0], a0, a1);
                    tc::f2_split(acc[1], b0, b1);
                    tc::f2_split(acc[2], c0, c1);
                    tc::f2_split(acc[3], d0, d1);
                    l += ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
                    continue;
                }
                const bool psplit = SDA_K2_PSPLIT && !spec;
                if (psplit) {
                    // every part but the last: its P into TMEM and announced before the next
                    // part's exponentials, so its PV overlaps the rest of the softmax
                    const float mu = (m_use == -INFINITY) ? 0.f : m_use;
                    constexpr int PP = 64 / kPParts;   // logit pairs per part
#pragma unroll
                    for (int part = 0; part < kPParts; ++part) {
                        exp_range(mu, false, mr0, mr1, part * PP, (part + 1) * PP);
                        if (part + 1 == kPParts) break;
                        if (PAIR) {
                            wait_pe();
#pragma unroll
                            for (int cc = part * PP / 4; cc < (part + 1) * PP / 4; ++cc) st_chunk(cc);
                            tc::fence_proxy_async_smem();
                        } else {
#pragma unroll
                            for (int c = part * PP / 8; c < (part + 1) * PP / 8; ++c) {
                                uint32_t pk[8];
#pragma unroll
                                for (int e = 0; e < 8; ++e)
                                    pk[e] = tc::pack_bf16(__uint_as_float(s[16 * c + 2 * e]), __uint_as_float(s[16 * c + 2 * e + 1]));
                                tc::tmem_st8(s_col + c * 8, pk);
                            }
                            tc::tmem_st_wait();
                        }
                        tc::tc_fence_before();
                        arrive0(&p_part[g * (kPParts - 1) + part]);
                    }
                } else if (!spec) {
                    exp_pass((m_use == -INFINITY) ? 0.f : m_use, false, mr0, mr1);
                } else if (__any_sync(0xffffffffu, need)) {
                    load_s();   // S is still in TMEM (P has not been written over it)
                    exp_pass(m_use, false, mr0, mr1);
                }
                uint64_t acc[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) acc[a] = tc::f2(0.f, 0.f);
#if SDA_K2_SUM_AFTER
                // P to TMEM first (packed 16 at a time; the fp32 values stay in s[]), the row sum
                // after the arrive: the FADD2 chains leave the softmax -> PV -> S chain
                if (PAIR) {
                    wait_pe();
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc) {
                        if (psplit && cc < (kPParts - 1) * 16 / kPParts) continue;   // already in SMEM
                        st_chunk(cc);
                    }
                    tc::fence_proxy_async_smem();
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (psplit && c < (kPParts - 1) * 8 / kPParts) continue;   // already in TMEM
                        uint32_t pk[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            pk[e] = tc::pack_bf16(__uint_as_float(s[16 * c + 2 * e]), __uint_as_float(s[16 * c + 2 * e + 1]));
                        tc::tmem_st8(s_col + c * 8, pk);
                    }
                    tc::tmem_st_wait();
                }
                tc::tc_fence_before();
                if ((warp & 3) == 0 && lane == 0) K2_STAMP(2 + g, j);
                if (!PAIR && g == 0 && (warp & 3) != 0 && lane == 0) K2_STAMP(17 + (warp & 3), j);   // warps 1-3: 18-20
                if (warp == 0 && lane == 0) K2_STAMP1(21, j);
#if SDA_K2_PSPLIT
                if (!psplit)   // (speculative path: whole P at once)
                    for (int part = 0; part + 1 < kPParts; ++part) arrive0(&p_part[g * (kPParts - 1) + part]);
#endif
                arrive0(&p_full[g]);
#pragma unroll
                for (int i = 0; i < 64; ++i)
                    acc[i & 3] = tc::fadd2(acc[i & 3], tc::f2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])));
#else
#pragma unroll
                for (int i = 0; i < 64; ++i) {
                    const float p0 = __uint_as_float(s[2 * i]), p1 = __uint_as_float(s[2 * i + 1]);
                    acc[i & 3] = tc::fadd2(acc[i & 3], tc::f2(p0, p1));
                    s[i] = tc::pack_bf16(p0, p1);
                }
#endif
                float a0, a1, b0, b1, c0, c1, d0, d1;
                tc::f2_split(acc[0], a0, a1);
                tc::f2_split(acc[1], b0, b1);
                tc::f2_split(acc[2], c0, c1);
                tc::f2_split(acc[3], d0, d1);
                l += ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
#if !SDA_K2_SUM_AFTER
#pragma unroll
                for (int c = 0; c < 8; ++c) tc::tmem_st8(s_col + c * 8, s + c * 8);
                tc::tmem_st_wait();
                tc::tc_fence_before();
                if ((warp & 3) == 0 && lane == 0) K2_STAMP(2 + g, j);
                tc::mbar_arrive(&p_full[g]);
#endif
            }
            if (HX) {
                if (group_live) {   // the helper's half of the row sum
                    asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
                    l += xch[2 * 2 * 2 * 128 + (segc & 1) * 256 + g * 128 + row];
                }
                ++segc;
            }
            // epilogue: O / l, (row_max, exp_sum) in natural units
            if (tid == 0) K2_STAMP(12, si_tr);
            const SoftKeep* const kk = opaque(keep);
            const Seg sg = kk->seg;
            const int64_t r_in = (int64_t)g * TILE + row;          // row within the unit
            const bool store = r_in < sg.nrows;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            const float st_max = l > 0.f ? m_run / kLog2e : -INFINITY;
            const float st_sum = l > 0.f ? l * ex2(m_use - m_run) : 0.f;
            if (p.sk) {
                // stream-K: a unit held whole by this CTA is written straight from TMEM (as in split
                // mode); a piece goes to this CTA's scratch slot, and the last of the unit's pieces
                // to finish merges them into the output
                const int T_sk = kk->T, NG = kk->NG, gq = p.sk_gq, qp_sk = (int)blockIdx.x % gq;
                const int g_a = sk_group_of(sg.ub, T_sk, NG);
                const int P = 1 + sk_group_of(sg.ub + sg.nt - 1, T_sk, NG) - g_a;   // pieces of the unit
                float* out_o = p.out_o;
                float* out_stats = p.out_stats;
                int64_t orow0 = sg.head_row;   // one split: output rows mirror the Q rows
                if (p.remote) {
                    float* rec = p.rec_peer[sg.b / p.b_per] + (sg.b % p.b_per) * p.rec_stride;
                    orow0 = sg.head_row - (int64_t)sg.b * p.q_heads * p.q_rows;
                    out_o = rec;
                    out_stats = rec + (int64_t)p.q_heads * p.q_rows * D;
                }
                // remote records are staged in slot 2 and copied out as whole 512-byte rows
                const bool direct = P == 1 && !p.remote;
                float* const slot2 = sk_slot(p, (int)blockIdx.x, 2);
                float* const slot = P == 1 ? slot2 : sk_slot(p, (int)blockIdx.x, sg.first ? 0 : 1);
                float* const dst_o = direct ? out_o + orow0 * D : slot;
                float* const dst_st = direct ? out_stats + orow0 * 2 : slot + 2 * TILE * D;
                if (group_live) {
                    if (warp_live) {
                        tc::mbar_wait(&o_final[g], oc & 1);
                        tc::tc_fence_after();
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            uint32_t o[16];
                            tc::tmem_ld16(o_col + c * 16, o);
                            tc::tmem_ld_wait();
                            if (store) store_row16(dst_o + r_in * D + c * 16, o, inv);
                        }
                    }
                    ++oc;
                    tc::tc_fence_before();
                    arrive0(&o_empty[g]);   // O_g may be overwritten by the next segment
                    if (store) *reinterpret_cast<float2*>(dst_st + r_in * 2) = make_float2(st_max, st_sum);
                }
                if (tid == 0) K2_STAMP(13, si_tr);
                if (direct) {
                    ++si_tr;
                    continue;
                }
                __threadfence();
                softmax_bar();
                if (tid == 0) {
                    uint32_t t = 0;
                    if (P > 1) {
                        t = atomicAdd(&p.sk_tick[sg.unit], 1u);
                        __threadfence();
                    }
                    *sk_ticket = t;
                }
                softmax_bar();
                if (tid == 0) K2_STAMP(14, si_tr);
                if ((int)*sk_ticket == P - 1) {
                    if (P > 1) {
                        // warp w merges rows 32w .. 32w+31: lane = row for the weights (from each
                        // piece's stats), then lanes across a row's 512 bytes for O' -- 16 rows
                        // (8 KB) in flight per warp, coalesced reads and writes. Piece k lives in
                        // CTA (group g_a + k, this pair): its first segment's slot unless that
                        // group's range starts before the unit.
                        __threadfence();
                        auto piece = [&](int k) -> const float* {
                            const int gk = g_a + k;
                            return sk_slot(p, gk * gq + qp_sk, sk_lo(T_sk, NG, gk) < sg.ub ? 1 : 0);
                        };
                        const int r_l = warp * 32 + lane;
                        const bool live_l = r_l < sg.nrows;
                        float mx = -INFINITY, L = 0.f;
                        for (int k = 0; k < P && live_l; ++k) {
                            const float2 stt = __ldcg(reinterpret_cast<const float2*>(piece(k) + 2 * TILE * D + r_l * 2));
                            if (stt.y > 0.f) mx = fmaxf(mx, stt.x);
                        }
                        for (int k = 0; k < P && live_l; ++k) {
                            const float2 stt = __ldcg(reinterpret_cast<const float2*>(piece(k) + 2 * TILE * D + r_l * 2));
                            if (stt.y > 0.f) L += stt.y * ex2((stt.x - mx) * kLog2e);
                        }
                        const float iv = L > 0.f ? 1.f / L : 0.f;
                        constexpr int MB = HX ? 8 : 16;   // rows per batch (split rows: 120 registers)
#pragma unroll 1
                        for (int h = 0; h < 32 / MB; ++h) {
                            const int rb = warp * 32 + h * MB;     // first row of this batch
                            float4 acc[MB];
#pragma unroll
                            for (int u = 0; u < MB; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                            for (int k = 0; k < P; ++k) {
                                const float* pk = piece(k);
                                float wl = 0.f;
                                if (live_l) {
                                    const float2 stt = __ldcg(reinterpret_cast<const float2*>(pk + 2 * TILE * D + r_l * 2));
                                    wl = stt.y > 0.f ? stt.y * ex2((stt.x - mx) * kLog2e) * iv : 0.f;
                                }
                                float4 v[MB];
#pragma unroll
                                for (int u = 0; u < MB; ++u)
                                    v[u] = rb + u < sg.nrows ? __ldcg(reinterpret_cast<const float4*>(pk + (rb + u) * D) + lane)
                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                                for (int u = 0; u < MB; ++u) {
                                    const float w = __shfl_sync(0xffffffffu, wl, h * MB + u);
                                    acc[u].x += w * v[u].x;
                                    acc[u].y += w * v[u].y;
                                    acc[u].z += w * v[u].z;
                                    acc[u].w += w * v[u].w;
                                }
                            }
#pragma unroll
                            for (int u = 0; u < MB; ++u)
                                if (rb + u < sg.nrows) reinterpret_cast<float4*>(out_o + (orow0 + rb + u) * D)[lane] = acc[u];
                        }
                        if (live_l) *reinterpret_cast<float2*>(out_stats + (orow0 + r_l) * 2) = make_float2(L > 0.f ? mx : -INFINITY, L);
                        if (p.remote) __threadfence_system();
                    } else if (p.remote) {
                        // one piece: slot 2 -> the inquirer's record, a warp per row, 4 rows in flight
                        softmax_bar();
                        for (int r = warp; r < sg.nrows; r += 32) {
                            float4 v[4];
                            float2 sv[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int rr = r + u * 8;
                                if (rr < sg.nrows) {
                                    v[u] = __ldcg(reinterpret_cast<const float4*>(slot2 + rr * D) + lane);
                                    sv[u] = __ldcg(reinterpret_cast<const float2*>(slot2 + 2 * TILE * D + rr * 2));
                                }
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int rr = r + u * 8;
                                if (rr < sg.nrows) {
                                    reinterpret_cast<float4*>(out_o + (orow0 + rr) * D)[lane] = v[u];
                                    if (lane == 0) *reinterpret_cast<float2*>(out_stats + (orow0 + rr) * 2) = sv[u];
                                }
                            }
                        }
                        __threadfence_system();
                    }
                    softmax_bar();
                    if (tid == 0) {
                        if (P > 1) p.sk_tick[sg.unit] = 0u;   // self-resetting for the next launch
                        if (p.remote) {   // the unit completing a destination's records raises its flag
                            const int64_t dest = sg.b / p.b_per;
                            const unsigned per_dest = (unsigned)((int64_t)p.q_heads * p.n_qpairs * p.b_per);
                            if (atomicAdd(&p.dest_counters[dest], 1u) == per_dest - 1) {
                                p.dest_counters[dest] = 0;
                                __threadfence_system();
                                flag_raise(p.peer_flag[dest], *p.epoch);
                            }
                        }
                    }
                }
                softmax_bar();   // scratch slot 2 and the ticket are reused by the next segment
                if (tid == 0) K2_STAMP(15, si_tr);
                ++si_tr;
                continue;
            }
            // split mode: output rows mirror the Q rows ([split][request][q head][q row])
            int64_t orow = (int64_t)sg.split * p.n_batch * p.q_heads * p.q_rows + sg.head_row + r_in;
            float* out_o = p.out_o;
            float* out_stats = p.out_stats;
            if (p.remote) {   // the packed record of request b in its inquirer's receive slot (one split)
                const int64_t dest = sg.b / p.b_per, i = sg.b % p.b_per;
                float* rec = p.rec_peer[dest] + i * p.rec_stride;
                orow = sg.head_row - (int64_t)sg.b * p.q_heads * p.q_rows + r_in;   // (head, row) within the request
                out_o = rec;
                out_stats = rec + (int64_t)p.q_heads * p.q_rows * D;
            }
            if (group_live && warp_live) {
                if (nkv > 0) {
                    tc::mbar_wait(&o_final[g], oc & 1);
                    tc::tc_fence_after();
                }
                // remote records: stage the warp's 32 rows in SMEM (group 0 reuses the K ring, whose
                // last reader has completed; group 1 the V ring) and write them as one contiguous
                // 16 KB run -- whole 512-byte rows per warp store instead of 32 scattered 16-byte
                // pieces, which NVLink carries far less efficiently
                // (rows of 512 B, 16-byte chunks XOR-swizzled by row & 7 against bank conflicts)
                // (the pair form does not run split-mode remote records: launch_k2_prefill_tc)
                float* stg = reinterpret_cast<float*>(smem + (g ? L::OFF_V : L::OFF_K) + (warp & 3) * 32 * 128 * 4);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint32_t o[16];
                    if (nkv > 0) {
                        tc::tmem_ld16(o_col + c * 16, o);
                        tc::tmem_ld_wait();
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = 0u;
                    }
                    if (p.remote) {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            *reinterpret_cast<float4*>(stg + lane * 128 + (((c * 4 + e) ^ (lane & 7)) * 4)) =
                                make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                            __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
                    } else if (store) {
                        store_row16(out_o + orow * D + c * 16, o, inv);
                    }
                }
                if (p.remote) {
                    __syncwarp();
                    // rows orow(lane 0) .. +31 are consecutive: 32 x 512 B contiguous (the tail of a
                    // partial tile stops at nrows)
                    const int64_t row0 = orow - lane;
                    const int nvalid = (int)min((int64_t)32, sg.nrows - (r_in - lane));
                    for (int r = 0; r < nvalid; ++r)
                        reinterpret_cast<float4*>(out_o + (row0 + r) * D)[lane] =
                            *reinterpret_cast<const float4*>(stg + r * 128 + ((lane ^ (r & 7)) * 4));
                }
                if (store) {
                    out_stats[orow * 2 + 0] = st_max;
                    out_stats[orow * 2 + 1] = st_sum;
                }
            }
            if (group_live && nkv > 0) {   // O_g may be overwritten by this CTA's next segment (causal pairs)
                ++oc;
                tc::tc_fence_before();
                arrive0(&o_empty[g]);
            }
        }
        if (p.sk) {
            // requests with no keys contribute no tiles: their units (zero O', stats (-inf, 0)) go
            // round-robin over the CTAs
            const int nq = p.n_qpairs;
            const int64_t upr = (int64_t)p.q_heads * nq;
            for (int64_t b = 0; b < p.n_batch; ++b) {
                if (ntile_of(p, b) != 0) continue;
                for (int64_t ui = 0; ui < upr; ++ui) {
                    if ((b * upr + ui) % gridDim.x != blockIdx.x) continue;
                    Seg z;
                    fill_unit(p, (int)b, (int)(ui / nq), (int)(ui % nq), z);
                    float* out_o = p.out_o;
                    float* out_stats = p.out_stats;
                    int64_t orow0 = z.head_row;
                    if (p.remote) {
                        float* rec = p.rec_peer[b / p.b_per] + (b % p.b_per) * p.rec_stride;
                        orow0 = z.head_row - b * p.q_heads * p.q_rows;
                        out_o = rec;
                        out_stats = rec + (int64_t)p.q_heads * p.q_rows * D;
                    }
                    for (int64_t r = warp; r < z.nrows; r += 8) {
                        reinterpret_cast<float4*>(out_o + (orow0 + r) * D)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (lane == 0) *reinterpret_cast<float2*>(out_stats + (orow0 + r) * 2) = make_float2(-INFINITY, 0.f);
                    }
                    if (p.remote) {
                        __threadfence_system();
                        softmax_bar();
                        if (tid == 0) {
                            const int64_t dest = b / p.b_per;
                            const unsigned per_dest = (unsigned)(upr * p.b_per);
                            if (atomicAdd(&p.dest_counters[dest], 1u) == per_dest - 1) {
                                p.dest_counters[dest] = 0;
                                __threadfence_system();
                                flag_raise(p.peer_flag[dest], *p.epoch);
                            }
                        }
                    }
                }
            }
        }
    }
    if (warp == 0) K2_CTA_STAMP(1);
    if (p.remote && !p.sk) __threadfence_system();   // this CTA's record stores visible system-wide
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (p.remote && !p.sk && tid == 0) {   // the CTA completing a destination's records raises its flag
        const int64_t dest = (int64_t)(blockIdx.z / p.n_splits) / p.b_per;
        const unsigned per_dest = gridDim.x * gridDim.y * (unsigned)(p.b_per * p.n_splits);
        if (atomicAdd(&p.dest_counters[dest], 1u) == per_dest - 1) {
            p.dest_counters[dest] = 0;
            __threadfence_system();
            flag_raise(p.peer_flag[dest], *p.epoch);
        }
    }
    if (PAIR) {
        tc::cluster_sync();   // the peer's MMAs (issued by rank 0) and TMEM reads are done
        if (warp == 0) tc::tmem_dealloc_pair<512>(tmem);
    } else if (warp == 0) {
        tc::tmem_dealloc<512>(tmem);
    }
}

bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);

// Normal mode for prefill spans (>= 64 rows per head); grouped mode for GQA decode, where the
// G q heads of a kv head (x a few rows) fill one 128-row tile and K/V are streamed once per group.
static bool k2_grouped(const K2Params& p) {
    const int64_t G = p.q_heads / p.kv_heads;
    return G > 1 && G * p.q_rows <= 128 && p.q_rows < 64;
}

bool k2_prefill_tc_eligible(const K2Params& p, int d, int qdt, int kvdt) {
    return d == 128 && qdt == SDA_BF16 && kvdt == SDA_BF16 && (p.q_rows >= 64 || k2_grouped(p));
}

// Stream-K layout of the caller's workspace: one ticket per unit first (the only part that must
// be zero; a launch leaves it zeroed), then 3 scratch slots per CTA from a 256-byte boundary.
namespace {
struct SkShape {
    int64_t gq;        // CTAs per group
    int64_t ctas;      // grid: groups x gq
    int64_t units;
    size_t tick_bytes;
    size_t bytes;      // 0: this shape does not run stream-K
};
SkShape sk_shape(int64_t n_batch, int q_heads, int64_t q_rows, int64_t kv_cap) {
    using namespace k2tc;
    SkShape s{1, 0, 0, 0, 0};
    const int64_t sms = device_sms();
    const int64_t nq = (q_rows + 2 * TILE - 1) / (2 * TILE);
    s.units = n_batch * q_heads * nq;
    const int64_t tiles_max = n_batch * q_heads * ((kv_cap + TILE - 1) / TILE);
    if (nq > sms || tiles_max >= (int64_t)INT32_MAX || s.units >= (int64_t)INT32_MAX || s.units == 0) return s;
    // CTAs per group: among the divisors of n_qpairs of at least min(4, n_qpairs) -- smaller
    // groups share each K/V tile between too few CTAs (C3: groups of 2, 482 us) -- the one that
    // leaves the fewest SMs idle, ties to the larger (C3: 37 groups of 4 = 148 SMs, 467 us,
    // against 18 groups of 8 = 144 SMs, 469-472 us)
    s.gq = nq;
    for (int64_t d = std::min<int64_t>(4, nq); d <= nq; ++d)
        if (nq % d == 0 && (sms / d) * d > (sms / s.gq) * s.gq) s.gq = d;
    if (const char* e = std::getenv("SDA_K2_SK_GQ")) {   // experiment override (must divide n_qpairs)
        const int64_t d = std::atoll(e);
        if (d >= 1 && d <= nq && nq % d == 0) s.gq = d;
    }
    const int64_t tiles_sub = tiles_max * (nq / s.gq);
    if (tiles_sub >= (int64_t)INT32_MAX) {
        s.bytes = 0;
        return s;
    }
    s.ctas = std::max<int64_t>(1, std::min<int64_t>(sms / s.gq, tiles_sub)) * s.gq;
    s.tick_bytes = ((size_t)s.units * sizeof(uint32_t) + 255) / 256 * 256;
    s.bytes = s.tick_bytes + (size_t)s.ctas * 3 * (size_t)SK_SLOT * sizeof(float);
    return s;
}
}  // namespace

size_t k2_prefill_sk_workspace_bytes(const K2Params& q) {
    if (k2_grouped(q)) return 0;
    return sk_shape(q.n_batch, q.q_heads, q.q_rows, q.kv_cap).bytes;
}

// the CTA-pair form as a cluster-of-2 launch
static cudaError_t launch_pair(dim3 grid, const K2TcParams& p, const CUtensorMap& qm, const CUtensorMap& km,
                               const CUtensorMap& vm, cudaStream_t st) {
    using namespace k2tc;
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k2_prefill_tc_kernel<true>), Lay<true>::SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(Thr<true>::N);
    cfg.dynamicSmemBytes = Lay<true>::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k2_prefill_tc_kernel<true>, p, qm, km, vm);
}

cudaError_t launch_k2_prefill_tc(const K2Params& q, cudaStream_t st) {
    using namespace k2tc;
    {
        const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k2_prefill_tc_kernel<false>), SMEM);
        if (e != cudaSuccess) return e;
    }
    K2TcParams p;
    p.q_rows = q.q_rows;
    p.kv_cap = q.kv_cap;
    p.kv_len = q.kv_len;
    p.out_o = q.out_o;
    p.out_stats = q.out_stats;
    p.n_batch = q.n_batch;
    p.q_heads = q.q_heads;
    p.kv_heads = q.kv_heads;
    p.n_splits = q.n_splits;
    p.grouped = k2_grouped(q) ? 1 : 0;
    p.n_qpairs = p.grouped ? 1 : (int)((q.q_rows + 2 * TILE - 1) / (2 * TILE));
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
    p.remote = q.remote_rec;
    p.b_per = q.b_per;
    p.rec_stride = q.rec_stride;
    for (int i = 0; i < kMaxPeers; ++i) {
        p.rec_peer[i] = static_cast<float*>(q.ll_rec[i]);
        p.peer_flag[i] = q.peer_flag[i];
    }
    p.dest_counters = q.dest_counters;
    p.epoch = q.epoch;
    p.sk = 0;
    p.sk_gq = 1;
    p.sk_buf = nullptr;
    p.sk_tick = nullptr;
    p.causal = q.causal ? 1 : 0;
    p.causal_offset = q.causal_offset;
    if (p.causal && p.grouped) return cudaErrorInvalidValue;
    CUtensorMap qm, km, vm, km64;
    if (!make_tmap_bf16_2d(&qm, q.q, q.n_batch * q.q_heads * q.q_rows, D, TILE) ||
        !make_tmap_bf16_2d(&km, q.k, q.n_batch * q.kv_heads * q.kv_cap, D, TILE) ||
        !make_tmap_bf16_2d(&vm, q.v, q.n_batch * q.kv_heads * q.kv_cap, D, TILE) ||
        !make_tmap_bf16_2d(&km64, q.k, q.n_batch * q.kv_heads * q.kv_cap, D, TILE / 2))
        return cudaErrorInvalidValue;
    // CTA pairs (opt-in, SDA_K2_PAIR=1; measured slower on C3): whole 256-row Q-tile
    // pairs everywhere, clusters of two CTAs that walk the same key tiles (stream-K groups of an
    // even size, or split mode's even pair count), no causal mask / grouped rows / split-mode
    // remote records
    const char* pe = std::getenv("SDA_K2_PAIR");
    const bool pair_ok = pe && pe[0] == '1' && !p.grouped && !p.causal && q.q_rows % (2 * TILE) == 0;
    // One split (not grouped) with the caller's workspace: stream-K over a persistent grid of
    // groups of n_qpairs CTAs, one CTA per SM, so the last wave is never partial (C3: 256 units
    // on 148 SMs ran as 2 waves, the second 73 % full).
    if (!p.grouped && !p.causal && q.n_splits == 1 && q.sk_work && !std::getenv("SDA_K2_NO_SK")) {
        const SkShape sh = sk_shape(q.n_batch, q.q_heads, q.q_rows, q.kv_cap);
        if (sh.bytes && q.sk_work_bytes >= sh.bytes) {
            p.sk = 1;
            p.sk_gq = (int)sh.gq;
            p.sk_tick = static_cast<uint32_t*>(q.sk_work);
            p.sk_buf = reinterpret_cast<float*>(static_cast<char*>(q.sk_work) + sh.tick_bytes);
            if (pair_ok && sh.gq % 2 == 0) return launch_pair(dim3((unsigned)sh.ctas), p, qm, km64, vm, st);
            k2_prefill_tc_kernel<false><<<dim3((unsigned)sh.ctas), Thr<false>::N, SMEM, st>>>(p, qm, km, vm);
            return cudaGetLastError();
        }
    }
    const dim3 grid = p.causal ? dim3((unsigned)q.q_heads, (unsigned)((p.n_qpairs + 1) / 2), (unsigned)(q.n_batch * q.n_splits))
                               : dim3((unsigned)p.n_qpairs, (unsigned)(p.grouped ? q.kv_heads : q.q_heads),
                                      (unsigned)(q.n_batch * q.n_splits));
    if (pair_ok && !p.remote && p.n_qpairs % 2 == 0) return launch_pair(grid, p, qm, km64, vm, st);
    k2_prefill_tc_kernel<false><<<grid, Thr<false>::N, SMEM, st>>>(p, qm, km, vm);
    return cudaGetLastError();
}

}  // namespace sda

#ifdef SDA_K2_TRACE
extern "C" int sda_debug_k2_trace(void* host) {
    return (int)cudaMemcpyFromSymbol(host, sda::g_k2_trace, sizeof(sda::g_k2_trace));
}
extern "C" int sda_debug_k2_cta(void* host) {
    return (int)cudaMemcpyFromSymbol(host, sda::g_k2_cta, sizeof(sda::g_k2_cta));
}
#endif
