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
// from HBM once per group instead of once per q head; 10 warps:
//   warp 8      TMA producer: Q0/Q1 once, then K_j / V_j tiles (128 keys) into 2-stage rings
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
};

#ifdef SDA_K2_TRACE
// debug build only (tools/k2_trace.py): globaltimer stamps of CTA (0,0,0) -- [kind][j], kinds:
// 0/1 softmax g got S, 2/3 softmax g arrives with P, 4/5 PV0/PV1 issue, 6/7 MMA loop top / V ready,
// 8 before the P1 wait, 9/10 before / after the K(j+1) wait
__device__ uint64_t g_k2_trace[16][64];
__device__ __forceinline__ void k2_stamp(int kind, int64_t j) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && j < 64) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_k2_trace[kind][j] = t;
    }
}
#define K2_STAMP(k, j) k2_stamp(k, j)
#else
#define K2_STAMP(k, j)
#endif

// The MMA warp's waits for P sit on the S -> softmax -> PV -> S chain of each Q tile: it spins
// (test_wait) instead of suspending (try_wait), which trims ~100 ns of wake-up per hand-off
// (tools/k2_trace.py; +2 % on C3).
#define K2_WAIT_P(b, ph) tc::mbar_wait_spin(b, ph)

namespace k2tc {
constexpr int D = 128;
constexpr int TILE = 128;
constexpr int TILE_BYTES = TILE * D * 2;          // 32 KB bf16 tile
constexpr int BLK = TILE * 128;                   // [128 x 64] swizzled block (16 KB)
constexpr int OFF_Q0 = 0, OFF_Q1 = OFF_Q0 + TILE_BYTES;
constexpr int OFF_K = OFF_Q1 + TILE_BYTES;        // 2 stages
constexpr int OFF_V = OFF_K + 2 * TILE_BYTES;     // 2 stages
constexpr int OFF_BAR = OFF_V + 2 * TILE_BYTES;
// barriers: q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[2], o_final[2]
constexpr int NBAR = 15;
constexpr int SMEM = OFF_BAR + NBAR * 8 + 16;
constexpr int THREADS = 320;
constexpr uint32_t COL_S0 = 0, COL_S1 = 128, COL_O0 = 256, COL_O1 = 384;
// Exponentials per 4 pairs computed on the FMA pipe (tc::exp2_fma2) instead of MUFU.EX2. Measured
// on C3 (exps batched ahead of the packing): 0 -> 489 us, 1 -> 485 us, 2 -> 547 us -- past one in
// four the added FMA-pipe instructions cost more issue time than the MUFU time they free.
#ifndef SDA_K2_EMU_OF4
#define SDA_K2_EMU_OF4 1
#endif
constexpr int kEmuOf4 = SDA_K2_EMU_OF4;
}  // namespace k2tc

__global__ void __launch_bounds__(320, 1)
k2_prefill_tc_kernel(const K2TcParams p, const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                     const __grid_constant__ CUtensorMap vmap) {
    using namespace k2tc;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* const bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* const q_full = bars;
    uint64_t* const k_full = bars + 1;
    uint64_t* const k_empty = bars + 3;
    uint64_t* const v_full = bars + 5;
    uint64_t* const v_empty = bars + 7;
    uint64_t* const s_full = bars + 9;
    uint64_t* const p_full = bars + 11;
    uint64_t* const o_final = bars + 13;
    uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // work unit: blockIdx.z = request * n_splits + split;
    //   normal : blockIdx.x = 256-row pair of Q tiles, blockIdx.y = q head
    //   grouped: blockIdx.y = kv head; the tile rows are its G q heads x Lq rows
    const int64_t b = blockIdx.z / p.n_splits;
    const int split = blockIdx.z % p.n_splits;
    const int G = p.q_heads / p.kv_heads;
    const int kvh = p.grouped ? (int)blockIdx.y : (int)blockIdx.y / G;
    const int64_t head_row = p.grouped ? (b * p.q_heads + (int64_t)kvh * G) * p.q_rows
                                       : (b * p.q_heads + blockIdx.y) * p.q_rows + (int64_t)blockIdx.x * 2 * TILE;
    const int64_t nrows = p.grouped ? (int64_t)G * p.q_rows
                                    : min((int64_t)2 * TILE, p.q_rows - (int64_t)blockIdx.x * 2 * TILE);
    const bool two = nrows > TILE;                  // second Q tile in use
    const int64_t len = p.kv_len ? (int64_t)p.kv_len[b] : p.kv_cap;
    // split ranges aligned to whole 128-key tiles
    const int64_t ntile_all = (len + TILE - 1) / TILE;
    const int64_t tps = (ntile_all + p.n_splits - 1) / p.n_splits;
    const int64_t t0 = (int64_t)split * tps;
    const int64_t t1 = min(ntile_all, t0 + tps);
    const int64_t nkv = t1 > t0 ? t1 - t0 : 0;
    const int64_t k_end = min(len, t1 * TILE);      // keys >= k_end are masked

    if (tid == 0) {
        tc::mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&k_full[i], 1);
            tc::mbar_init(&k_empty[i], 1);
            tc::mbar_init(&v_full[i], 1);
            tc::mbar_init(&v_empty[i], 1);
            tc::mbar_init(&s_full[i], 1);
            tc::mbar_init(&p_full[i], 128);
            tc::mbar_init(&o_final[i], 1);
        }
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int64_t qrow0 = head_row;                       // global row of this CTA's first Q row
    const int64_t kvrow0 = ((b * p.kv_heads + kvh) * p.kv_cap) + t0 * TILE;

    if (warp == 8) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0 && nkv > 0) {
            tc::prefetch_tmap(&qmap);
            tc::prefetch_tmap(&kmap);
            tc::prefetch_tmap(&vmap);
            tc::mbar_arrive_expect_tx(q_full, (two ? 2 : 1) * TILE_BYTES);
            for (int g = 0; g < (two ? 2 : 1); ++g)
                for (int kb = 0; kb < 2; ++kb)
                    tc::tma_load_2d(smem + (g ? OFF_Q1 : OFF_Q0) + kb * BLK, &qmap, kb * 64, (int)(qrow0 + g * TILE), q_full);
            for (int64_t j = 0; j < nkv; ++j) {
                const int st = (int)(j & 1);
                const uint32_t ph = (uint32_t)(((j >> 1) - 1) & 1);
                if (j >= 2) tc::mbar_wait(&k_empty[st], ph);
                tc::mbar_arrive_expect_tx(&k_full[st], TILE_BYTES);
                for (int kb = 0; kb < 2; ++kb)
                    tc::tma_load_2d(smem + OFF_K + st * TILE_BYTES + kb * BLK, &kmap, kb * 64, (int)(kvrow0 + j * TILE), &k_full[st]);
                if (j >= 2) tc::mbar_wait(&v_empty[st], ph);
                tc::mbar_arrive_expect_tx(&v_full[st], TILE_BYTES);
                for (int kb = 0; kb < 2; ++kb)
                    tc::tma_load_2d(smem + OFF_V + st * TILE_BYTES + kb * BLK, &vmap, kb * 64, (int)(kvrow0 + j * TILE), &v_full[st]);
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------------------------ MMA issuer
        // the whole warp runs the loop (warp-uniform descriptors); the elected lane issues
        if (nkv > 0) {
            const bool leader = tc::elect_one();
            constexpr uint32_t IDESC_S = tc::idesc_bf16_f32(128, 128, false, false);   // Q K^T, both K-major
            constexpr uint32_t IDESC_O = tc::idesc_bf16_f32(128, 128, false, true);    // P V, V MN-major
            const uint32_t q0 = tc::smem_u32(smem + OFF_Q0), q1 = tc::smem_u32(smem + OFF_Q1);
            const uint32_t kbase = tc::smem_u32(smem + OFF_K), vbase = tc::smem_u32(smem + OFF_V);
            auto issue_s = [&](int g, int64_t j) {
                const int st = (int)(j & 1);
                const uint32_t qa = g ? q1 : q0;
                const uint32_t kb = kbase + st * TILE_BYTES;
                const uint32_t d_tmem = tmem + (g ? COL_S1 : COL_S0);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t off = (k >> 2) * BLK + (k & 3) * 32;
                    const uint64_t da = tc::sw128_desc(qa + off, 16, 1024), db = tc::sw128_desc(kb + off, 16, 1024);
                    if (leader) tc::mma_bf16_ss(d_tmem, da, db, IDESC_S, k > 0 ? 1u : 0u);
                }
                if (leader) tc::mma_commit(&s_full[g]);
            };
            auto issue_pv = [&](int g, int64_t j) {
                const int st = (int)(j & 1);
                const uint32_t vb = vbase + st * TILE_BYTES;
                const uint32_t d_tmem = tmem + (g ? COL_O1 : COL_O0);
                const uint32_t p_tmem = tmem + (g ? COL_S1 : COL_S0);
#pragma unroll
                for (int k = 0; k < TILE / 16; ++k) {   // 16 keys per step: P columns 8k.., V rows 16k..
                    const uint64_t db = tc::sw128_desc(vb + k * 2048, BLK, 1024);
                    if (leader) tc::mma_bf16_ts(d_tmem, p_tmem + k * 8, db, IDESC_O, (j > 0 || k > 0) ? 1u : 0u);
                }
            };
            tc::mbar_wait(q_full, 0);
            tc::mbar_wait(&k_full[0], 0);
            tc::tc_fence_after();
            issue_s(0, 0);
            if (two) issue_s(1, 0);
            if (leader) tc::mma_commit(&k_empty[0]);
            for (int64_t j = 0; j < nkv; ++j) {
                const int st = (int)(j & 1);
                const uint32_t ph = (uint32_t)((j >> 1) & 1);
                K2_STAMP(6, j);
                tc::mbar_wait(&v_full[st], ph);
                K2_STAMP(7, j);
                K2_WAIT_P(&p_full[0], (uint32_t)(j & 1));
                tc::tc_fence_after();
                K2_STAMP(4, j);
                issue_pv(0, j);
                if (!two && leader) tc::mma_commit(&v_empty[st]);
                if (j + 1 == nkv && leader) tc::mma_commit(&o_final[0]);
                if (j + 1 < nkv) {
                    const int sn = (int)((j + 1) & 1);
                    K2_STAMP(9, j);
                    tc::mbar_wait(&k_full[sn], (uint32_t)(((j + 1) >> 1) & 1));
                    K2_STAMP(10, j);
                    tc::tc_fence_after();
                    issue_s(0, j + 1);
                    if (!two && leader) tc::mma_commit(&k_empty[sn]);
                }
                if (!two) continue;
                K2_STAMP(8, j);
                K2_WAIT_P(&p_full[1], (uint32_t)(j & 1));
                tc::tc_fence_after();
                K2_STAMP(5, j);
                issue_pv(1, j);
                if (leader) tc::mma_commit(&v_empty[st]);
                if (j + 1 == nkv && leader) tc::mma_commit(&o_final[1]);
                if (j + 1 < nkv) {
                    issue_s(1, j + 1);
                    if (leader) tc::mma_commit(&k_empty[(j + 1) & 1]);
                }
            }
        }
    } else {
        // ------------------------------------------------------------------ softmax groups
        const int g = warp >> 2;                               // Q tile
        const int row = (warp & 3) * 32 + lane;                // TMEM lane = tile row
        const int64_t tile_row0 = (int64_t)g * TILE + (warp & 3) * 32;
        const bool group_live = g == 0 || two;
        // warps whose 32 rows are all past the CTA's rows only keep the barrier protocol going
        const bool warp_live = tile_row0 < nrows;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t s_col = tmem + (g ? COL_S1 : COL_S0) + lane_off;
        const uint32_t o_col = tmem + (g ? COL_O1 : COL_O0) + lane_off;
        float m_run = -INFINITY, m_use = -INFINITY, l = 0.f;
        for (int64_t j = 0; group_live && j < nkv; ++j) {
            tc::mbar_wait(&s_full[g], (uint32_t)(j & 1));
            tc::tc_fence_after();
            if ((warp & 3) == 0 && lane == 0) K2_STAMP(g, j);
            if (!warp_live) {
                tc::tc_fence_before();
                tc::mbar_arrive(&p_full[g]);
                continue;
            }
            uint32_t s[128];
#pragma unroll
            for (int c = 0; c < 8; ++c) tc::tmem_ld16(s_col + c * 16, s + c * 16);
            tc::tmem_ld_wait();
            const int64_t valid = k_end - (t0 + j) * TILE;      // keys of this tile still in range
            if (valid < TILE) {                                   // only the split's last tile
#pragma unroll
                for (int i = 0; i < 128; ++i)
                    if (i >= valid) s[i] = 0xFF800000u;           // -inf
            }
            // row max on the raw logits (scale > 0), two new values per 3-input max (splitting the
            // TMEM load to overlap the max measured slower)
            float mr0 = -INFINITY, mr1 = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; i += 2) {
                mr0 = tc::fmax3(mr0, __uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1]));
                mr1 = tc::fmax3(mr1, __uint_as_float(s[2 * i + 2]), __uint_as_float(s[2 * i + 3]));
            }
            const float mt = fmaxf(mr0, mr1) * p.scale_log2;
            const float m_new = fmaxf(m_run, mt);
            m_run = m_new;
            // lazy rescale: keep the exponent base unless the max grew by more than 8 (x256)
            const bool need = m_new > m_use + 8.f;
            if (__any_sync(0xffffffffu, need && j > 0 && m_use > -INFINITY)) {
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
            const float mu = (m_use == -INFINITY) ? 0.f : m_use;
            // p = exp2(s * scale - mu) in place (one packed FFMA2 per two logits), all 128 first:
            // the MUFU ops issue back to back instead of each waiting on its consumer; then the row
            // sum (4 packed FADD2 chains) and the bf16x2 packing of P in place (s[i] <- p[2i], p[2i+1])
            const uint64_t sc2 = tc::f2(p.scale_log2, p.scale_log2), nmu2 = tc::f2(-mu, -mu);
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                float x0, x1;
                tc::f2_split(tc::ffma2(tc::f2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sc2, nmu2), x0, x1);
                float p0, p1;
                if ((i & 3) < kEmuOf4) {
                    tc::exp2_fma2(x0, x1, p0, p1);
                } else {
                    p0 = ex2(x0);
                    p1 = ex2(x1);
                }
                s[2 * i] = __float_as_uint(p0);
                s[2 * i + 1] = __float_as_uint(p1);
            }
            uint64_t acc[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) acc[a] = tc::f2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                const float p0 = __uint_as_float(s[2 * i]), p1 = __uint_as_float(s[2 * i + 1]);
                acc[i & 3] = tc::fadd2(acc[i & 3], tc::f2(p0, p1));
                s[i] = tc::pack_bf16(p0, p1);
            }
            float a0, a1, b0, b1, c0, c1, d0, d1;
            tc::f2_split(acc[0], a0, a1);
            tc::f2_split(acc[1], b0, b1);
            tc::f2_split(acc[2], c0, c1);
            tc::f2_split(acc[3], d0, d1);
            l += ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
#pragma unroll
            for (int c = 0; c < 8; ++c) tc::tmem_st8(s_col + c * 8, s + c * 8);
            tc::tmem_st_wait();
            tc::tc_fence_before();
            if ((warp & 3) == 0 && lane == 0) K2_STAMP(2 + g, j);
            tc::mbar_arrive(&p_full[g]);
        }
        // epilogue: O / l, (row_max, exp_sum) in natural units
        const int64_t r_in = (int64_t)g * TILE + row;          // row within this CTA's rows
        const bool store = r_in < nrows;
        // output rows mirror the Q rows ([split][request][q head][q row]); head_row already holds
        // request, head and row-tile offsets
        int64_t orow = (int64_t)split * p.n_batch * p.q_heads * p.q_rows + head_row + r_in;
        float* out_o = p.out_o;
        float* out_stats = p.out_stats;
        if (p.remote) {   // the packed record of request b in its inquirer's receive slot (one split)
            const int64_t dest = b / p.b_per, i = b % p.b_per;
            float* rec = p.rec_peer[dest] + i * p.rec_stride;
            orow = head_row - b * p.q_heads * p.q_rows + r_in;   // (head, row) within the request
            out_o = rec;
            out_stats = rec + (int64_t)p.q_heads * p.q_rows * D;
        }
        if (group_live && warp_live) {
            if (nkv > 0) {
                tc::mbar_wait(&o_final[g], 0);
                tc::tc_fence_after();
            }
            const float inv = l > 0.f ? 1.f / l : 0.f;
            // remote records: stage the warp's 32 rows in SMEM (group 0 reuses the K ring, whose
            // last reader has completed; group 1 the V ring) and write them as one contiguous
            // 16 KB run -- whole 512-byte rows per warp store instead of 32 scattered 16-byte
            // pieces, which NVLink carries far less efficiently
            // (rows of 512 B, 16-byte chunks XOR-swizzled by row & 7 against bank conflicts)
            float* stg = reinterpret_cast<float*>(smem + (g ? OFF_V : OFF_K) + (warp & 3) * 32 * 128 * 4);
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
                    float4* dst = reinterpret_cast<float4*>(out_o + orow * D + c * 16);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        dst[e] = make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                             __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
                }
            }
            if (p.remote) {
                __syncwarp();
                // rows orow(lane 0) .. +31 are consecutive: 32 x 512 B contiguous (the tail of a
                // partial tile stops at nrows)
                const int64_t row0 = orow - lane;
                const int nvalid = (int)min((int64_t)32, nrows - (r_in - lane));
                for (int r = 0; r < nvalid; ++r)
                    reinterpret_cast<float4*>(out_o + (row0 + r) * D)[lane] =
                        *reinterpret_cast<const float4*>(stg + r * 128 + ((lane ^ (r & 7)) * 4));
            }
            if (store) {
                const bool any = l > 0.f;
                out_stats[orow * 2 + 0] = any ? m_run / kLog2e : -INFINITY;
                out_stats[orow * 2 + 1] = any ? l * ex2(m_use - m_run) : 0.f;
            }
        }
    }
    if (p.remote) __threadfence_system();   // this CTA's record stores visible system-wide
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (p.remote && tid == 0) {   // the CTA completing a destination's records raises its flag
        const int64_t dest = b / p.b_per;
        const unsigned per_dest = gridDim.x * gridDim.y * (unsigned)(p.b_per * p.n_splits);
        if (atomicAdd(&p.dest_counters[dest], 1u) == per_dest - 1) {
            p.dest_counters[dest] = 0;
            __threadfence_system();
            flag_raise(p.peer_flag[dest], *p.epoch);
        }
    }
    if (warp == 0) tc::tmem_dealloc<512>(tmem);
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

cudaError_t launch_k2_prefill_tc(const K2Params& q, cudaStream_t st) {
    using namespace k2tc;
    {
        const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k2_prefill_tc_kernel), SMEM);
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
    CUtensorMap qm, km, vm;
    if (!make_tmap_bf16_2d(&qm, q.q, q.n_batch * q.q_heads * q.q_rows, D, TILE) ||
        !make_tmap_bf16_2d(&km, q.k, q.n_batch * q.kv_heads * q.kv_cap, D, TILE) ||
        !make_tmap_bf16_2d(&vm, q.v, q.n_batch * q.kv_heads * q.kv_cap, D, TILE))
        return cudaErrorInvalidValue;
    const dim3 grid((unsigned)p.n_qpairs, (unsigned)(p.grouped ? q.kv_heads : q.q_heads),
                    (unsigned)(q.n_batch * q.n_splits));
    k2_prefill_tc_kernel<<<grid, THREADS, SMEM, st>>>(p, qm, km, vm);
    return cudaGetLastError();
}

}  // namespace sda

#ifdef SDA_K2_TRACE
extern "C" int sda_debug_k2_trace(void* host) {
    return (int)cudaMemcpyFromSymbol(host, sda::g_k2_trace, sizeof(sda::g_k2_trace));
}
#endif
