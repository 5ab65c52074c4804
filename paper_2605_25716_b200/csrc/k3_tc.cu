// k3_tc.cu -- K3 on the 5th-generation tensor cores for prefill-shaped merges: LSE-weighted merge
// of one domain's K2 splits (+ plaintext sources), inverse token permutation and the phi_V^-1
// unscramble as a tcgen05 GEMM against an exact +-1 bf16 sign matrix.
//
// Replaces, per output row, dec_output (scrambler.cpp:138-149: O = scatter_rows(O' phi_V^-1, p_q))
// followed by merge_shards (attention.cpp:89-123), as span_finish_layer composes them
// (protocol.cpp:926-948) -- the same contract as k3_merge.cu's warp forms, which stay the path for
// decode rows, LL sources, quantised wires and merges over several key groups.
//
// With the key image's tables (which = 1, phi_V): for an output row,
//   y[i] = InvOut[i] * sum_m (-1)^popcount(P1[i] & P2^-1[m]) * InvIn[m] * acc[m]
// (u[j] = t[P2[j]], w = H u, y[i] = w[P1[i]] InvOut[i] with t = acc InvIn, as the warp forms run
// it), acc = sum_s w_s O'_s[p_q^-1[r]] over the group's splits. So Y = (acc o InvIn) B^T o InvOut
// with B[i][m] = (-1)^popcount(P1[i] & P2^-1[m]) exact in bf16. The f32 rows t = acc o InvIn are
// split exactly into three bf16 parts (hi + mid + lo carry all 24 significand bits), so
// D = t_hi B^T + t_mid B^T + t_lo B^T in the f32 TMEM accumulator is t B^T up to the accumulator's
// own rounding -- no bf16 rounding of the data anywhere.
//
// Per CTA (persistent, one per SM, a contiguous run of 128-row tiles of (request, head) slabs),
// warp-specialised, 12 warps:
//   warps 4-11 (split)   : a warp per row, a lane per d/32 columns: coalesced loads of the rows
//                          O'_s[p_q^-1[r]] of every split, the weighted sum, o InvIn, the exact
//                          3-way bf16 split into a SWIZZLE_128B K-major A stage (two stages);
//                          split warp 0 then issues the tile's 3 x d/16 tcgen05.mma (M=128, N=d,
//                          K=16) into one of two TMEM accumulators (tcgen05.commit);
//   warps 0-3  (epilogue): tcgen05.ld (a thread per row) -> f32 rows into the finished A stage,
//                          then a warp per row: o InvOut, + the plaintext sources' weighted rows
//                          (the inquirer's own span, natural row order), / the LSE denominator,
//                          coalesced stores of the output rows and stats; they also build B when
//                          the (request, key head) changes.
// HBM-bound: 4d + 8 bytes read per (row, source), d * sizeof(out) written per row; the GEMM is
// 3 x 2 x 128 x d x d flop per tile (~50 flop per byte at d = 128).
#include "common.cuh"
#include "tc_util.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace sda {

// Debug timeline (SDA_K3TC_TRACE=1): clock64 stamps of one split warp and one epilogue warp per
// CTA, read back with sda_debug_k3tc_trace (tools/k3_trace.py).
constexpr int kK3TraceSlots = 64;
__device__ unsigned long long g_k3tc_trace[256][kK3TraceSlots];   // persistent grids: <= one CTA per SM

struct K3TcArgs {
    K3Params p;
    int nk, np;              // keyed sources (one key group) and plaintext sources (<= 1)
    int kidx[SDA_MAX_SOURCES];
    int pidx;
    int64_t ntr;             // 128-row tiles per (request, head)
    int64_t total_tiles;
    int64_t tiles_per_cta;
    int trace;
};

template <int D>
struct K3TcShape {
    static constexpr int TILE = 128;
    static constexpr int V = D / 32;                  // columns per lane in the row-per-warp phases
    static constexpr int BLK = TILE * 128;            // one [128 x 64] bf16 SW128 block of A
    static constexpr int PART = TILE * D * 2;         // one bf16 part of an A tile
    static constexpr int ABUF = 3 * PART;             // hi, mid, lo
    static constexpr int BBLK = D * 128;              // one [D x 64] bf16 SW128 block of B
    static constexpr int OFF_A = 0;                   // 2 x ABUF
    static constexpr int OFF_B = 2 * ABUF;
    static constexpr int OFF_RI = OFF_B + D * D * 2;  // [2][128] {1/denominator, plaintext weight}
    static constexpr int OFF_BAR = OFF_RI + 2 * TILE * 8;
    static constexpr int SMEM = OFF_BAR + 64;
    static constexpr uint32_t TMEM_COLS = 2 * D;
    static constexpr int SPLIT_WARPS = 8;
    static constexpr int ROWS_PER_SPLIT = TILE / SPLIT_WARPS;   // 16
    static constexpr int THREADS = 32 * (4 + SPLIT_WARPS);
};

// byte offset of 16-byte chunk q of row r in the f32 staging rows (D * 4 bytes each): the low
// three bits of q are XOR-ed with r so both the thread-per-row writes and the warp-per-row reads
// are bank-conflict-free
template <int D>
__device__ __forceinline__ uint32_t stg_off(uint32_t r, uint32_t q) {
    return r * (D * 4) + (((q & ~7u) | ((q & 7u) ^ (r & 7u))) << 4);
}

template <int V>
__device__ __forceinline__ void ldg_vec(const float* p, float* v) {
    if constexpr (V == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
    } else {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = t.x, v[1] = t.y;
    }
}

// A CTA's position in its run of tiles: (request, head) slab, key slab and first row, advanced one
// tile at a time (no divisions past the first).
struct K3Tile {
    uint32_t bh, b, h, kslab;
    int64_t row0;
};

template <int D, typename TOut, int NK>
__global__ void __launch_bounds__(384, 1) k3_tc_kernel(const __grid_constant__ K3TcArgs a) {
    using S = K3TcShape<D>;
    constexpr int V = S::V, RPS = S::ROWS_PER_SPLIT;
    constexpr int RB = 4 / NK;    // rows per split-warp batch; a ring of four batches, three in flight
    constexpr int NB = RPS / RB;  // batches per tile (a multiple of 4)
    static_assert(NK <= 2 && NB % 4 == 0, "batches rotate through four register sets");
    // bf16 parts of t: hi + mid + lo is exact (f32 output); hi + mid carries 16 significant bits
    // (~2^-17 relative), far below the bf16 output's own rounding
    constexpr int NPART = std::is_same<TOut, float>::value ? 3 : 2;
    const K3Params& p = a.p;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* const abuf = smem + S::OFF_A;
    uint8_t* const bmat = smem + S::OFF_B;
    float2* const rinfo = reinterpret_cast<float2*>(smem + S::OFF_RI);
    uint64_t* const afull = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
    uint64_t* const afree = afull + 2;
    uint64_t* const tfull = afree + 2;
    uint64_t* const bready = tfull + 2;
    uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(bready + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    auto stamp = [&](int slot) {
        if (a.trace && lane == 0 && slot < kK3TraceSlots && blockIdx.x < 256) g_k3tc_trace[blockIdx.x][slot] = clock64();
    };
    const int64_t first = (int64_t)blockIdx.x * a.tiles_per_cta;
    const int64_t last = min(first + a.tiles_per_cta, a.total_tiles);
    if (first >= last) return;
    const int64_t ntiles = last - first;
    const uint32_t H = (uint32_t)p.q_heads, G = (uint32_t)(p.q_heads / p.key_heads);
    const uint8_t* const keys = p.src[a.kidx[0]].keys;
    const bool single = p.n_src == 1;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&afull[i], S::SPLIT_WARPS);
            tc::mbar_init(&afree[i], 4);
            tc::mbar_init(&tfull[i], 1);
        }
        tc::mbar_init(bready, 128);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();   // launched early behind K2 (PDL): its partials must be complete
    if (warp == 0) stamp(0);

    auto tile_at = [&](int64_t it) {
        K3Tile t;
        const uint32_t id = (uint32_t)(first + it), ntr = (uint32_t)a.ntr;
        t.bh = id / ntr;
        t.row0 = (int64_t)(id - t.bh * ntr) * S::TILE;
        t.b = t.bh / H;
        t.h = t.bh - t.b * H;
        t.kslab = t.b * (uint32_t)p.key_heads + t.h / G;
        return t;
    };
    auto advance = [&](K3Tile& t) {
        t.row0 += S::TILE;
        if (t.row0 >= p.q_rows) {
            t.row0 = 0;
            ++t.bh;
            if (++t.h == H) {
                t.h = 0;
                ++t.b;
            }
            t.kslab = t.b * (uint32_t)p.key_heads + t.h / G;
        }
    };
    // element offset of slab (b, h) in a source laid out [.., q_rows, per_row]
    auto src_off = [&](const K3Source& s, const K3Tile& t, int per_row) -> int64_t {
        return s.bstride ? (int64_t)t.b * s.bstride + (int64_t)t.h * p.q_rows * per_row
                         : (int64_t)t.bh * p.q_rows * per_row;
    };

    if (warp >= 4) {
        // ------------------------------------------------------------------ split warps
        // Rows sw*16 .. sw*16+15 of every tile. Lane j < 16 prepares row j of a tile ahead of its
        // use in three stages (p_q^-1 index, then stats, then weights), so no dependent load sits
        // on the critical path; the O' rows stream in batches of RB rows, two batches in flight.
        const int sw = warp - 4;
        const int jr = lane & 15;
        auto load_ridx = [&](int64_t it, const K3Tile& t, uint32_t (&r)[NK]) {
#pragma unroll
            for (int k = 0; k < NK; ++k) r[k] = 0;
            const int64_t rowj = t.row0 + sw * RPS + jr;
            if (it >= ntiles || rowj >= p.q_rows) return;
#pragma unroll
            for (int k = 0; k < NK; ++k)
                if (k < a.nk) {
                    const uint32_t* pq = p.src[a.kidx[k]].pq_inv;
                    r[k] = pq ? __ldg(pq + (int64_t)t.b * p.pq_bstride + rowj) : (uint32_t)rowj;
                }
        };
        auto load_stats = [&](int64_t it, const K3Tile& t, const uint32_t (&r)[NK], float2 (&st)[NK], float2& stp) {
#pragma unroll
            for (int k = 0; k < NK; ++k) st[k] = make_float2(-INFINITY, 0.f);
            stp = make_float2(-INFINITY, 0.f);
            const int64_t rowj = t.row0 + sw * RPS + jr;
            if (it >= ntiles || rowj >= p.q_rows) return;
#pragma unroll
            for (int k = 0; k < NK; ++k)
                if (k < a.nk) {
                    const K3Source& s = p.src[a.kidx[k]];
                    st[k] = __ldg(reinterpret_cast<const float2*>(s.stats + src_off(s, t, 2)) + r[k]);
                }
            if (a.np) {
                const K3Source& s = p.src[a.pidx];
                stp = __ldg(reinterpret_cast<const float2*>(s.stats + src_off(s, t, 2)) + rowj);
            }
        };
        // merge weights of a row (attention.cpp:103-121); a dead source (exp_sum 0) gets w < 0
        struct Wts {
            float w[NK];
            float wp, mstar, denom;
        };
        auto weights = [&](const float2 (&st)[NK], const float2& stp) {
            Wts o;
            o.mstar = -INFINITY;
#pragma unroll
            for (int k = 0; k < NK; ++k)
                if (st[k].y > 0.f) o.mstar = fmaxf(o.mstar, st[k].x);
            if (stp.y > 0.f) o.mstar = fmaxf(o.mstar, stp.x);
            o.denom = 0.f;
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const bool live = st[k].y > 0.f;
                const float w = live ? (single ? 1.f : st[k].y * expf(st[k].x - o.mstar)) : 0.f;
                o.denom += single ? st[k].y : w;
                o.w[k] = live ? w : -1.f;
            }
            const float wp = stp.y > 0.f ? stp.y * expf(stp.x - o.mstar) : 0.f;
            o.denom += wp;
            o.wp = stp.y > 0.f ? wp : -1.f;
            return o;
        };
        // the O' rows of RB rows (row q*RB + j of this warp's 16 in tile t, indices r)
        auto issue = [&](const K3Tile& t, int q, const uint32_t (&r)[NK], float (&x)[RB][NK][V]) {
            const float* ob[NK];
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const K3Source& s = p.src[a.kidx[k < a.nk ? k : 0]];
                ob[k] = s.o + src_off(s, t, D) + lane * V;
            }
            // unconditional loads straight into x: rows past q_rows read row 0 (index 0) and unused
            // source slots read source 0, both under a weight < 0 -- no select after a load, so
            // nothing waits on it before its use
#pragma unroll
            for (int j = 0; j < RB; ++j)
#pragma unroll
                for (int k = 0; k < NK; ++k)
                    ldg_vec<V>(ob[k] + (int64_t)__shfl_sync(0xffffffffu, r[k], q * RB + j) * D, x[j][k]);
        };
        const int c0 = lane * V;   // this lane's first column
        const uint32_t aoff = (c0 / 64) * S::BLK + ((c0 % 8) * 2);
        const uint32_t chunk = (c0 % 64) / 8;
        float inin[V];
        auto compute = [&](int q, const Wts& wt, const float (&x)[RB][NK][V], uint8_t* A) {
#pragma unroll
            for (int j = 0; j < RB; ++j) {
                float acc[V];
#pragma unroll
                for (int e = 0; e < V; ++e) acc[e] = 0.f;
#pragma unroll
                for (int k = 0; k < NK; ++k) {
                    const float w = __shfl_sync(0xffffffffu, wt.w[k], q * RB + j);
                    if (w >= 0.f)   // never 0 * NaN for a dead split (or a padding slot / row)
#pragma unroll
                        for (int e = 0; e < V; ++e) acc[e] = fmaf(w, x[j][k][e], acc[e]);
                }
                // t = acc / s2, split exactly: t = hi + mid + lo (bf16 each)
                uint32_t hw[V / 2], mw[V / 2], lw[V / 2];
#pragma unroll
                for (int e = 0; e < V; e += 2) {
                    const float t0 = __fmul_rn(acc[e], inin[e]), t1 = __fmul_rn(acc[e + 1], inin[e + 1]);
                    float h0, h1, m0, m1;
                    hw[e / 2] = tc::pack_bf16(t0, t1);
                    bf16x2_to_f2(hw[e / 2], h0, h1);
                    const float r0 = __fsub_rn(t0, h0), r1 = __fsub_rn(t1, h1);
                    mw[e / 2] = tc::pack_bf16(r0, r1);
                    if constexpr (NPART == 3) {
                        bf16x2_to_f2(mw[e / 2], m0, m1);
                        lw[e / 2] = tc::pack_bf16(__fsub_rn(r0, m0), __fsub_rn(r1, m1));
                    }
                }
                const uint32_t off = aoff + tc::sw128_off((uint32_t)(sw * RPS + q * RB + j), chunk);
                if constexpr (V == 4) {
                    *reinterpret_cast<uint2*>(A + off) = make_uint2(hw[0], hw[1]);
                    *reinterpret_cast<uint2*>(A + S::PART + off) = make_uint2(mw[0], mw[1]);
                    if constexpr (NPART == 3) *reinterpret_cast<uint2*>(A + 2 * S::PART + off) = make_uint2(lw[0], lw[1]);
                } else {
                    *reinterpret_cast<uint32_t*>(A + off) = hw[0];
                    *reinterpret_cast<uint32_t*>(A + S::PART + off) = mw[0];
                    if constexpr (NPART == 3) *reinterpret_cast<uint32_t*>(A + 2 * S::PART + off) = lw[0];
                }
            }
        };
        // prep pipeline: c = tile it (weights ready), b = tile it+1 (stats in flight),
        // a = tile it+2 (p_q^-1 in flight); tile cursors tc_ .. t3 = it .. it+3
        K3Tile tc_ = tile_at(0), t1 = tc_, t2, t3;
        advance(t1);
        t2 = t1;
        advance(t2);
        t3 = t2;
        advance(t3);
        uint32_t ridx_c[NK], ridx_b[NK], ridx_a[NK];
        float2 st_b[NK], stp_b;
        load_ridx(0, tc_, ridx_c);
        load_ridx(1, t1, ridx_b);
        load_ridx(2, t2, ridx_a);
        float x0[RB][NK][V], x1[RB][NK][V], x2[RB][NK][V], x3[RB][NK][V];
        // the first O' rows as soon as their indices arrive (NB >= 4: batches 0-2 are tile 0's)
        issue(tc_, 0, ridx_c, x0);
        issue(tc_, 1, ridx_c, x1);
        issue(tc_, 2, ridx_c, x2);
        load_stats(0, tc_, ridx_c, st_b, stp_b);
        Wts wc = weights(st_b, stp_b);
        load_stats(1, t1, ridx_b, st_b, stp_b);
        uint32_t cur = 0xffffffffu, mma_slab = 0xffffffffu, nbuild = 0;
        constexpr uint32_t IDESC = tc::idesc_bf16_f32(128, D, false, false);
#pragma unroll 1
        for (int64_t it = 0; it < ntiles; ++it) {
            const int bi = (int)(it & 1);
            const bool more = it + 1 < ntiles;
            if (tc_.kslab != cur) {
                const float* ft =
                    reinterpret_cast<const float*>(scrambler_ptr(keys, p.keys_bstride, tc_.b, (int)(tc_.h / G), D, 1));
                ldg_vec<V>(ft + kInvIn * D + lane * V, inin);
                cur = tc_.kslab;
            }
            uint8_t* const A = abuf + bi * S::ABUF;
            // batch q + 3 (this tile's, or the next tile's first ones) into the ring slot batch
            // q - 1 just left, then batch q
            // (unconditional -- past the CTA's last tile it re-reads valid rows -- so the loads land
            // in the ring registers directly, not in temporaries moved over on a branch join)
            auto ahead = [&](int q, float (&x)[RB][NK][V]) {
                const bool same = q + 3 < NB || !more;
                uint32_t r[NK];
#pragma unroll
                for (int k = 0; k < NK; ++k) r[k] = same ? ridx_c[k] : ridx_b[k];
                issue(same ? tc_ : t1, same ? (q + 3) % NB : q + 3 - NB, r, x);
            };
#pragma unroll 1
            for (int q = 0; q < NB; q += 4) {
                ahead(q, x3);
                if (q == 0) {
                    if (sw == 0 && it < 7) stamp(2 + 8 * (int)it);
                    if (it >= 2) tc::mbar_wait(&afree[bi], (uint32_t)(((it >> 1) - 1) & 1));
                    if (sw == 0 && it < 7) stamp(3 + 8 * (int)it);
                    // this tile's per-row merge results: for the epilogue, and out_stats / err
                    const int64_t rowj = tc_.row0 + sw * RPS + jr;
                    if (lane < 16 && rowj < p.q_rows) {
                        const bool masked = !(wc.mstar > -INFINITY);
                        const float inv = masked ? __int_as_float(0x7fc00000) : (single ? 1.f : 1.f / wc.denom);
                        rinfo[bi * S::TILE + sw * RPS + lane] = make_float2(inv, wc.wp);
                        if (masked && p.err) atomicExch(p.err, (int32_t)SDA_ERR_MASKED_ROW);
                        if (p.out_stats) {
                            float* sbh = p.out_stats + (p.out_bstride ? (int64_t)tc_.b * p.out_bstride + (int64_t)tc_.h * p.q_rows * 2
                                                                      : (int64_t)tc_.bh * p.q_rows * 2);
                            *reinterpret_cast<float2*>(sbh + rowj * 2) = make_float2(
                                single ? (masked ? -INFINITY : wc.mstar) : wc.mstar, masked ? 0.f : wc.denom);
                        }
                    }
                }
                compute(q, wc, x0, A);
                ahead(q + 1, x0);
                compute(q + 1, wc, x1, A);
                ahead(q + 2, x1);
                compute(q + 2, wc, x2, A);
                ahead(q + 3, x2);
                compute(q + 3, wc, x3, A);
            }
            tc::fence_proxy_async_smem();   // generic-proxy stores -> tcgen05 (async proxy) reads
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&afull[bi]);
            if (sw == 0 && it < 7) stamp(4 + 8 * (int)it);
            if (sw == 0) {   // the tile's MMAs, once every split warp has written its rows
                if (tc_.kslab != mma_slab) {
                    tc::mbar_wait(bready, nbuild & 1);   // the epilogue built this slab's B
                    ++nbuild;
                    mma_slab = tc_.kslab;
                }
                tc::mbar_wait(&afull[bi], (uint32_t)((it >> 1) & 1));
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(bi * D);
                const uint32_t asm_ = tc::smem_u32(A), bsm = tc::smem_u32(bmat);
                if (tc::elect_one()) {
#pragma unroll
                    for (int part = 0; part < NPART; ++part)
#pragma unroll
                        for (int k = 0; k < D / 16; ++k) {
                            const uint32_t ao = part * S::PART + (k >> 2) * S::BLK + (k & 3) * 32;
                            const uint32_t bo = (k >> 2) * S::BBLK + (k & 3) * 32;
                            tc::mma_bf16_ss(d_tmem, tc::sw128_desc(asm_ + ao, 16, 1024),
                                            tc::sw128_desc(bsm + bo, 16, 1024), IDESC, (part | k) ? 1u : 0u);
                        }
                    tc::mma_commit(&tfull[bi]);
                }
                __syncwarp();
                if (it < 7) stamp(5 + 8 * (int)it);
            }
            // advance the prep pipeline by one tile
            wc = weights(st_b, stp_b);
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                ridx_c[k] = ridx_b[k];
                ridx_b[k] = ridx_a[k];
            }
            tc_ = t1;
            t1 = t2;
            t2 = t3;
            advance(t3);
            load_stats(it + 2, t1, ridx_b, st_b, stp_b);
            load_ridx(it + 3, t2, ridx_a);
        }
    } else {
        // ------------------------------------------------------------------ epilogue (+ B build)
        // Tile by tile: tcgen05.ld of the accumulator, the merge epilogue, the output stores; when
        // the key slab changes (the previous tile finished, so its MMAs are done) B is rebuilt first.
        const int row = tid;   // TMEM lane = tile row in the thread-per-row phase
        float inout[V];
        constexpr int CPR = D / 8;   // 16-byte chunks per B row; a thread keeps one chunk column
        const int bc = tid % CPR;
        auto build_b = [&](const K3Tile& t) {
            const uint8_t* sc = scrambler_ptr(keys, p.keys_bstride, t.b, (int)(t.h / G), D, 1);
            const uint16_t* ut = reinterpret_cast<const uint16_t*>(sc + kU16Off * D);
            uint32_t p2i[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) p2i[j] = ut[kP2Inv * D + 8 * bc + j];
            ldg_vec<V>(reinterpret_cast<const float*>(sc) + kInvOut * D + lane * V, inout);
            // B[n][m] = (-1)^popcount(P1[n] & P2^-1[m]): row n = output column, K-major
#pragma unroll 4
            for (int i = 0; i < D * CPR / 128; ++i) {
                const int n = tid / CPR + i * (128 / CPR);
                const uint32_t pn = ut[kP1 * D + n];
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t s0 = __popc(pn & p2i[2 * j]) & 1, s1 = __popc(pn & p2i[2 * j + 1]) & 1;
                    w[j] = (s0 ? 0xBF80u : 0x3F80u) | ((s1 ? 0xBF80u : 0x3F80u) << 16);
                }
                *reinterpret_cast<uint4*>(bmat + (bc >> 3) * S::BBLK + tc::sw128_off(n, bc & 7)) =
                    make_uint4(w[0], w[1], w[2], w[3]);
            }
            tc::fence_proxy_async_smem();   // B (generic stores) -> tcgen05 reads
            tc::mbar_arrive(bready);
            if (warp == 0) stamp(1);
        };
        auto finish = [&](int64_t it, const K3Tile& t) {
            const int bi = (int)(it & 1);
            const float* pbase = a.np ? p.src[a.pidx].o + src_off(p.src[a.pidx], t, D) + lane * V : nullptr;
            const int64_t prow0 = t.row0 + warp * 32;
            // plaintext rows (the inquirer's own span, natural order) of this warp's 32, eight at
            // a time; rows past q_rows read row 0 (their results are not stored)
            constexpr int RB2 = 8;
            auto load_plain = [&](int j0, float (&xp)[RB2][V]) {
                if (a.np) {
#pragma unroll
                    for (int j = 0; j < RB2; ++j) {
                        const int64_t rg = prow0 + j0 + j;
                        ldg_vec<V>(pbase + (rg < p.q_rows ? rg : 0) * D, xp[j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < RB2; ++j)
#pragma unroll
                        for (int e = 0; e < V; ++e) xp[j][e] = 0.f;
                }
            };
            float xpa[RB2][V], xpb[RB2][V];
            load_plain(0, xpa);
            // phase 1: accumulator row (thread per row) -> f32 staging in this tile's A stage
            if (warp == 0 && it < 7) stamp(6 + 8 * (int)it);
            tc::mbar_wait(&tfull[bi], (uint32_t)((it >> 1) & 1));
            tc::tc_fence_after();
            if (warp == 0 && it < 7) stamp(7 + 8 * (int)it);
            uint8_t* const stg = abuf + bi * S::ABUF;
            constexpr int LDS_PER_WAIT = D / 16 < 4 ? D / 16 : 4;   // 64 columns per tcgen05.wait
#pragma unroll
            for (int c0 = 0; c0 < D / 16; c0 += LDS_PER_WAIT) {
                uint32_t r[LDS_PER_WAIT][16];
#pragma unroll
                for (int c = 0; c < LDS_PER_WAIT; ++c)
                    tc::tmem_ld16(tmem_base + (uint32_t)(bi * D + (c0 + c) * 16) + ((uint32_t)(warp * 32) << 16), r[c]);
                tc::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < LDS_PER_WAIT; ++c)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<uint4*>(stg + stg_off<D>(row, (c0 + c) * 4 + q)) =
                            make_uint4(r[c][4 * q], r[c][4 * q + 1], r[c][4 * q + 2], r[c][4 * q + 3]);
            }
            tc::tc_fence_before();
            __syncwarp();
            if (warp == 0 && it < 7) stamp(9 + 8 * (int)it);
            // phase 2: a warp per row over this warp's 32 rows: o InvOut, + plaintext, / denom
            TOut* const obh = static_cast<TOut*>(p.out) + (p.out_bstride ? (int64_t)t.b * p.out_bstride + (int64_t)t.h * p.q_rows * D
                                                                          : (int64_t)t.bh * p.q_rows * D);
            // all eight rows' staging reads first, then the arithmetic, then the stores (rows past
            // q_rows computed but not stored): no per-row branch serialising the loads
            auto rows8 = [&](int j0, const float (&xp)[RB2][V]) {
                float2 ri[RB2];
                float y[RB2][V];
#pragma unroll
                for (int j = 0; j < RB2; ++j) {
                    const int r = warp * 32 + j0 + j;
                    ri[j] = rinfo[bi * S::TILE + r];
                    if constexpr (V == 4) {
                        const float4 v4 = *reinterpret_cast<const float4*>(stg + stg_off<D>(r, lane));
                        y[j][0] = v4.x, y[j][1] = v4.y, y[j][2] = v4.z, y[j][3] = v4.w;
                    } else {
                        const float2 v2 = *reinterpret_cast<const float2*>(stg + stg_off<D>(r, lane >> 1) + (lane & 1) * 8);
                        y[j][0] = v2.x, y[j][1] = v2.y;
                    }
                }
#pragma unroll
                for (int j = 0; j < RB2; ++j)
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        float v = __fmul_rn(y[j][e], inout[e]);
                        if (ri[j].y >= 0.f) v = fmaf(ri[j].y, xp[j][e], v);
                        y[j][e] = v * ri[j].x;
                    }
#pragma unroll
                for (int j = 0; j < RB2; ++j) {
                    const int64_t rg = prow0 + j0 + j;
                    if (rg < p.q_rows) store_vec_any<V>(obh + rg * D + lane * V, y[j]);
                }
            };
            // the plaintext rows of the next eight in flight while these eight are finished (the
            // first eight were requested before the accumulator wait)
            load_plain(8, xpb);
            rows8(0, xpa);
            load_plain(16, xpa);
            rows8(8, xpb);
            load_plain(24, xpb);
            rows8(16, xpa);
            rows8(24, xpb);
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&afree[bi]);
            if (warp == 0 && it < 7) stamp(8 + 8 * (int)it);
        };
        K3Tile t = tile_at(0);
        uint32_t cur = 0xffffffffu;
#pragma unroll 1
        for (int64_t it = 0; it < ntiles; ++it) {
            if (t.kslab != cur) {   // tile it-1 is finished, so its MMAs are done: B is free
                build_b(t);
                cur = t.kslab;
            }
            finish(it, t);
            advance(t);
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem_base);
}

template <int D, typename TOut, int NK>
static cudaError_t launch_k3_tc_t(K3TcArgs& a, cudaStream_t st) {
    using S = K3TcShape<D>;
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k3_tc_kernel<D, TOut, NK>), S::SMEM);
    if (e != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>(a.total_tiles, device_sms());
    a.tiles_per_cta = (a.total_tiles + grid - 1) / grid;
    const int64_t ngrid = (a.total_tiles + a.tiles_per_cta - 1) / a.tiles_per_cta;
    return pdl_launch_smem(k3_tc_kernel<D, TOut, NK>, dim3((unsigned)ngrid), dim3(S::THREADS), S::SMEM, st, a);
}

template <int D, typename TOut>
static cudaError_t launch_k3_tc_d(K3TcArgs& a, cudaStream_t st) {
    if (a.nk == 1) return launch_k3_tc_t<D, TOut, 1>(a, st);
    return launch_k3_tc_t<D, TOut, 2>(a, st);
}

// The tensor-core form takes plain-memory, unquantised merges of d 64 / 128 with >= 128 rows per
// (request, head) whose keyed sources form ONE key group (a domain's splits) plus at most one
// plaintext source; anything else returns cudaErrorNotSupported and goes to the warp forms.
cudaError_t launch_k3_tc(const K3Params& p, int d, int odt, cudaStream_t st) {
    if (p.ll || p.quant_bits > 0 || (d != 64 && d != 128) || p.q_rows < 128 || p.n_src < 1 || p.n_src > SDA_MAX_SOURCES)
        return cudaErrorNotSupported;
    K3TcArgs a{};
    a.p = p;
    const uint8_t* keys = nullptr;
    for (int s = 0; s < p.n_src; ++s) {
        if (p.src[s].keys) {
            if (keys && p.src[s].keys != keys) return cudaErrorNotSupported;   // several key groups
            keys = p.src[s].keys;
            a.kidx[a.nk++] = s;
        } else {
            if (a.np == 1) return cudaErrorNotSupported;
            a.pidx = s;
            a.np = 1;
        }
        // 16-byte row loads (8 at d = 64): the ABI's alignment check guarantees them
    }
    // 3+ splits of the group: the warp forms' preload kernel is as fast (tools/k3_bench.py)
    if (a.nk == 0 || a.nk > 2) return cudaErrorNotSupported;
    a.trace = getenv("SDA_K3TC_TRACE") != nullptr;
    a.ntr = (p.q_rows + 127) / 128;
    a.total_tiles = a.ntr * p.n_batch * p.q_heads;
    if (a.total_tiles == 0) return cudaSuccess;
    if (a.total_tiles >= (int64_t(1) << 31)) return cudaErrorNotSupported;   // 32-bit tile ids
    const bool bf = odt == SDA_BF16;
    if (d == 64) return bf ? launch_k3_tc_d<64, __nv_bfloat16>(a, st) : launch_k3_tc_d<64, float>(a, st);
    return bf ? launch_k3_tc_d<128, __nv_bfloat16>(a, st) : launch_k3_tc_d<128, float>(a, st);
}

}  // namespace sda

// debug: the last traced launch's per-CTA clock64 stamps (n_cta x 64)
extern "C" int sda_debug_k3tc_trace(unsigned long long* host, int n_cta) {
    if (n_cta > 256) n_cta = 256;
    return cudaMemcpyFromSymbol(host, sda::g_k3tc_trace, sizeof(unsigned long long) * sda::kK3TraceSlots * n_cta) ==
                   cudaSuccess
               ? 0
               : 1;
}
