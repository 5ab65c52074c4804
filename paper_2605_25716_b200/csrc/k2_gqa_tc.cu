// k2_gqa_tc.cu -- K2 for GQA decode on tcgen05: keyless partial attention of the G query heads
// that share a kv head, with keys on the MMA M dimension ("swapped" flash decoding).
//
// Replaces shard_attention(q', K', V', none) (attention.cpp:42-78) for delegated decode with
// grouped heads (BASELINE config 5: 64 q heads / 8 kv heads). GQA is not in the reference
// (SPEC.md:310); the key rule is the reference's with head tag = kv head.
//
// Decode is HBM-bound: every K/V byte must be read once per (request, kv head), then used by
// all G heads (8 flop/B at G=8 -- beyond SIMT FMA throughput, trivial for tensor cores). The
// R = G x L_q query rows (<= 32) are the MMA N dimension and 128 keys the M dimension:
//   S^T[128 keys x N] = K_j . Q^T          (A = K tile, K-major; B = Q, K-major)
//   O^T[128 d x N]   += V_j^T . P^T         (A = V tile, MN-major; B = P^T in SMEM, K-major)
// so a tile's softmax is spread over 128 threads (one key each, R values per thread) instead of
// R threads. Per-head maxima are reduced across the CTA (shuffles + SMEM); running sums stay
// per thread (every thread uses the same exponent base) and are reduced once at the end; O^T
// is rescaled lazily (only when a head's max grows by more than 2^8).
// One CTA per (request, kv head, split), 6 warps: 0-3 softmax/epilogue, 4 TMA producer
// (3-stage K/V ring), 5 MMA issuer.
#include <cmath>

#include "common.cuh"
#include "tc_util.cuh"

namespace sda {

struct K2GqaParams {
    int64_t q_rows;
    int64_t kv_cap;
    const int32_t* kv_len;
    float* out_o;
    float* out_stats;
    int64_t n_batch;
    int q_heads;
    int kv_heads;
    int n_splits;
    int rows;              // R = G * q_rows (real rows of the N dimension)
    float scale_log2;
    // LL exchange (decode, q_rows == 1; epoch != nullptr): split `split` of request b = (dest, i)
    // is written as LL record rows [d O' | row_max, exp_sum] at logical float
    // ((split * b_per + i) * q_heads + head) * (d + 2) of ll_rec[dest] (as k2_decode.cu)
    const uint32_t* epoch;
    int64_t b_per;
    void* ll_rec[kMaxPeers];
};

namespace k2g {
constexpr int D = 128, TILE = 128, ST = 3;
constexpr int TILE_BYTES = TILE * D * 2;   // 32 KB
constexpr int BLK = TILE * 128;            // [128 x 64] swizzled block
template <int N>
struct Shape {
    static constexpr int Q_BYTES = N * D * 2;             // 2 K-blocks of [N x 64]
    static constexpr int QBLK = N * 128;
    static constexpr int P_BYTES = N * TILE * 2;          // P^T [N x 128 keys], 2 K-blocks
    static constexpr int OFF_K = 0;
    static constexpr int OFF_V = OFF_K + ST * TILE_BYTES;
    static constexpr int OFF_Q = OFF_V + ST * TILE_BYTES;
    static constexpr int OFF_P = OFF_Q + Q_BYTES;         // 2 buffers
    static constexpr int OFF_RED = OFF_P + 2 * P_BYTES;   // f32 [4 warps][N] per-warp maxima
    static constexpr int OFF_BAR = OFF_RED + 4 * N * 4 + 64;
    static constexpr int NBAR = 1 + 2 * ST + 2 + 2 + 2 + 2;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16;
    static constexpr uint32_t TMEM_COLS = 3 * N <= 64 ? 64 : 128;   // S^T x2, O^T
};
}  // namespace k2g

template <int N>
__global__ void __launch_bounds__(192, 1)
k2_gqa_tc_kernel(const K2GqaParams p, const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ CUtensorMap vmap) {
    using namespace k2g;
    using S = Shape<N>;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* const bars = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
    uint64_t* const q_full = bars;
    uint64_t* const kv_full = bars + 1;
    uint64_t* const kv_empty = bars + 1 + ST;
    uint64_t* const s_full = bars + 1 + 2 * ST;
    uint64_t* const p_full = s_full + 2;
    uint64_t* const p_free = p_full + 2;
    uint64_t* const pv_done = p_free + 2;
    uint64_t* const o_final = pv_done + 1;
    uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(bars + S::NBAR);
    float* const red = reinterpret_cast<float*>(smem + S::OFF_RED);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kvh = blockIdx.y;
    const int64_t b = blockIdx.z / p.n_splits;
    const int split = blockIdx.z % p.n_splits;
    const int G = p.q_heads / p.kv_heads;
    const int64_t len = p.kv_len ? (int64_t)p.kv_len[b] : p.kv_cap;
    const int64_t ntile_all = (len + TILE - 1) / TILE;
    const int64_t tps = (ntile_all + p.n_splits - 1) / p.n_splits;
    const int64_t t0 = (int64_t)split * tps;
    const int64_t t1 = min(ntile_all, t0 + tps);
    const int64_t nkv = t1 > t0 ? t1 - t0 : 0;
    const int64_t k_end = min(len, t1 * TILE);
    const int64_t qrow0 = (b * p.q_heads + (int64_t)kvh * G) * p.q_rows;   // first of the R Q rows
    const uint32_t ep = p.epoch ? *p.epoch : 0u;
    if (p.epoch) pdl_trigger();   // K3 may launch once every CTA has read the epoch
    const int64_t kvrow0 = (b * p.kv_heads + kvh) * p.kv_cap + t0 * TILE;

    if (tid == 0) {
        tc::mbar_init(q_full, 1);
        for (int i = 0; i < ST; ++i) {
            tc::mbar_init(&kv_full[i], 1);
            tc::mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&s_full[i], 1);
            tc::mbar_init(&p_full[i], 128);
            tc::mbar_init(&p_free[i], 1);
        }
        tc::mbar_init(pv_done, 1);
        tc::mbar_init(o_final, 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t COL_S = 0, COL_O = 2 * N;   // S^T buffers at [0, N), [N, 2N); O^T at [2N, 3N)

    if (warp == 4) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0 && nkv > 0) {
            tc::prefetch_tmap(&qmap);
            tc::prefetch_tmap(&kmap);
            tc::prefetch_tmap(&vmap);
            tc::mbar_arrive_expect_tx(q_full, S::Q_BYTES);
            for (int kb = 0; kb < 2; ++kb)
                tc::tma_load_2d(smem + S::OFF_Q + kb * S::QBLK, &qmap, kb * 64, (int)qrow0, q_full);
            for (int64_t j = 0; j < nkv; ++j) {
                const int st = (int)(j % ST);
                if (j >= ST) tc::mbar_wait(&kv_empty[st], (uint32_t)(((j / ST) - 1) & 1));
                tc::mbar_arrive_expect_tx(&kv_full[st], 2 * TILE_BYTES);
                for (int kb = 0; kb < 2; ++kb) {
                    tc::tma_load_2d(smem + S::OFF_K + st * TILE_BYTES + kb * BLK, &kmap, kb * 64, (int)(kvrow0 + j * TILE),
                                    &kv_full[st]);
                    tc::tma_load_2d(smem + S::OFF_V + st * TILE_BYTES + kb * BLK, &vmap, kb * 64, (int)(kvrow0 + j * TILE),
                                    &kv_full[st]);
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------------ MMA issuer
        // the whole warp runs the loop (warp-uniform descriptors); the elected lane issues
        if (nkv > 0) {
            const bool leader = tc::elect_one();
            constexpr uint32_t IDESC_S = tc::idesc_bf16_f32(128, N, false, false);  // K . Q^T
            constexpr uint32_t IDESC_O = tc::idesc_bf16_f32(128, N, true, false);   // V^T (MN-major) . P^T
            const uint32_t qb = tc::smem_u32(smem + S::OFF_Q);
            auto issue_s = [&](int64_t j) {
                const int st = (int)(j % ST);
                const uint32_t kb = tc::smem_u32(smem + S::OFF_K + st * TILE_BYTES);
                const uint32_t d_tmem = tmem + COL_S + (uint32_t)((j & 1) * N);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint64_t da = tc::sw128_desc(kb + (k >> 2) * BLK + (k & 3) * 32, 16, 1024);
                    const uint64_t db = tc::sw128_desc(qb + (k >> 2) * S::QBLK + (k & 3) * 32, 16, 1024);
                    if (leader) tc::mma_bf16_ss(d_tmem, da, db, IDESC_S, k > 0 ? 1u : 0u);
                }
                if (leader) tc::mma_commit(&s_full[j & 1]);
            };
            tc::mbar_wait(q_full, 0);
            for (int64_t j = 0; j < nkv && j < 2; ++j) {
                tc::mbar_wait(&kv_full[j % ST], 0);
                tc::tc_fence_after();
                issue_s(j);
            }
            for (int64_t j = 0; j < nkv; ++j) {
                const int st = (int)(j % ST);
                tc::mbar_wait(&p_full[j & 1], (uint32_t)((j >> 1) & 1));
                tc::tc_fence_after();
                const uint32_t vb = tc::smem_u32(smem + S::OFF_V + st * TILE_BYTES);
                const uint32_t pb = tc::smem_u32(smem + S::OFF_P + (j & 1) * S::P_BYTES);
#pragma unroll
                for (int k = 0; k < TILE / 16; ++k) {   // 16 keys per step
                    const uint64_t da = tc::sw128_desc(vb + k * 2048, BLK, 1024);
                    const uint64_t db = tc::sw128_desc(pb + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024);
                    if (leader) tc::mma_bf16_ss(tmem + COL_O, da, db, IDESC_O, (j > 0 || k > 0) ? 1u : 0u);
                }
                if (leader) {
                    tc::mma_commit(&kv_empty[st]);
                    tc::mma_commit(&p_free[j & 1]);
                    tc::mma_commit(pv_done);
                    if (j + 1 == nkv) tc::mma_commit(o_final);
                }
                if (j + 2 < nkv) {
                    tc::mbar_wait(&kv_full[(j + 2) % ST], (uint32_t)(((j + 2) / ST) & 1));
                    tc::tc_fence_after();
                    issue_s(j + 2);
                }
            }
        }
    } else {
        // ------------------------------------------------------------------ softmax (thread = key)
        const int R = p.rows;
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        float m_run[N], m_use[N], l[N];
#pragma unroll
        for (int h = 0; h < N; ++h) {
            m_run[h] = -INFINITY;
            m_use[h] = -INFINITY;
            l[h] = 0.f;
        }
        for (int64_t j = 0; j < nkv; ++j) {
            tc::mbar_wait(&s_full[j & 1], (uint32_t)((j >> 1) & 1));
            tc::tc_fence_after();
            uint32_t sv[N];
#pragma unroll
            for (int c = 0; c < N / 16; ++c) tc::tmem_ld16(tmem + COL_S + (uint32_t)((j & 1) * N + c * 16) + lane_off, sv + c * 16);
            tc::tmem_ld_wait();
            const bool valid = (t0 + j) * TILE + tid < k_end;
            float x[N];
#pragma unroll
            for (int h = 0; h < N; ++h) x[h] = valid ? __uint_as_float(sv[h]) * p.scale_log2 : -INFINITY;
            // per-head tile max over the 128 keys of the CTA
            float wm[N];
#pragma unroll
            for (int h = 0; h < N; ++h) {
                float v = x[h];
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                wm[h] = v;
            }
            if (lane == 0) {
#pragma unroll
                for (int h = 0; h < N; ++h) red[warp * N + h] = wm[h];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            bool any_rescale = false;
            float alpha[N];
#pragma unroll
            for (int h = 0; h < N; ++h) {
                const float tm = fmaxf(fmaxf(red[h], red[N + h]), fmaxf(red[2 * N + h], red[3 * N + h]));
                const float mn = fmaxf(m_run[h], tm);
                m_run[h] = mn;
                alpha[h] = 1.f;
                if (mn > m_use[h] + 8.f) {
                    if (m_use[h] > -INFINITY) {
                        alpha[h] = ex2(m_use[h] - mn);
                        any_rescale = true;
                    }
                    m_use[h] = mn;
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");   // `red` may be rewritten next tile
            if (any_rescale) {   // CTA-uniform: every thread holds the same maxima
                if (j > 0) {
                    tc::mbar_wait(pv_done, (uint32_t)((j - 1) & 1));   // PV(j-1) finished writing O^T
                    tc::tc_fence_after();
                }
                uint32_t ov[N];
#pragma unroll
                for (int c = 0; c < N / 16; ++c) tc::tmem_ld16(tmem + COL_O + (uint32_t)(c * 16) + lane_off, ov + c * 16);
                tc::tmem_ld_wait();
#pragma unroll
                for (int h = 0; h < N; ++h) {
                    ov[h] = __float_as_uint(__uint_as_float(ov[h]) * alpha[h]);
                    l[h] *= alpha[h];
                }
#pragma unroll
                for (int c = 0; c < N / 8; ++c) tc::tmem_st8(tmem + COL_O + (uint32_t)(c * 8) + lane_off, ov + c * 8);
                tc::tmem_st_wait();
            }
            // P^T[h][key] in bf16, K-major SW128 (key = this thread's row of the tile)
            if (j >= 2) tc::mbar_wait(&p_free[j & 1], (uint32_t)(((j >> 1) - 1) & 1));
            uint8_t* pbuf = smem + S::OFF_P + (j & 1) * S::P_BYTES + (tid >> 6) * (N * 128);
            const int kk = tid & 63;
#pragma unroll
            for (int h = 0; h < N; ++h) {
                const float pv = (h < R && m_use[h] > -INFINITY) ? ex2(x[h] - m_use[h]) : 0.f;
                l[h] += pv;
                *reinterpret_cast<__nv_bfloat16*>(pbuf + tc::sw128_off(h, kk >> 3) + (kk & 7) * 2) = __float2bfloat16_rn(pv);
            }
            tc::fence_proxy_async_smem();
            tc::tc_fence_before();
            tc::mbar_arrive(&p_full[j & 1]);
        }
        // ---- epilogue: l reduced over the CTA; O^T lane = d index, column = row
        float lt[N];
#pragma unroll
        for (int h = 0; h < N; ++h) {
            float v = l[h];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            lt[h] = v;
        }
        if (lane == 0) {
#pragma unroll
            for (int h = 0; h < N; ++h) red[warp * N + h] = lt[h];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
        for (int h = 0; h < N; ++h) lt[h] = red[h] + red[N + h] + red[2 * N + h] + red[3 * N + h];
        uint32_t ov[N];
        if (nkv > 0) {
            tc::mbar_wait(o_final, 0);
            tc::tc_fence_after();
#pragma unroll
            for (int c = 0; c < N / 16; ++c) tc::tmem_ld16(tmem + COL_O + (uint32_t)(c * 16) + lane_off, ov + c * 16);
            tc::tmem_ld_wait();
        } else {
#pragma unroll
            for (int h = 0; h < N; ++h) ov[h] = 0u;
        }
        if (p.epoch) {   // LL records straight into the inquirer's slot (q_rows == 1: row = q head)
            const int64_t dest = b / p.b_per, i = b % p.b_per;
            uint8_t* rb = static_cast<uint8_t*>(p.ll_rec[dest]) +
                          8 * (((int64_t)split * p.b_per + i) * p.q_heads + (int64_t)kvh * G) * (D + 2);
#pragma unroll
            for (int h = 0; h < N; ++h) {
                const float inv = lt[h] > 0.f ? 1.f / lt[h] : 0.f;
                const float o_here = __uint_as_float(ov[h]) * inv;               // d = tid
                const float o_next = __shfl_down_sync(0xffffffffu, o_here, 1);  // d = tid + 1
                if (h < R) {
                    uint8_t* row = rb + 8 * ((int64_t)h * (D + 2));
                    if ((tid & 1) == 0) ll_store(row + 8 * tid, __float_as_uint(o_here), __float_as_uint(o_next), ep);
                    if (tid == 0) {
                        const bool any = lt[h] > 0.f;
                        ll_store(row + 8 * D, __float_as_uint(any ? m_run[h] / kLog2e : -INFINITY),
                                 __float_as_uint(any ? lt[h] * ex2(m_use[h] - m_run[h]) : 0.f), ep);
                    }
                }
            }
        }
        const int64_t orow0 = (int64_t)split * p.n_batch * p.q_heads * p.q_rows + qrow0;
#pragma unroll
        for (int h = 0; h < N && !p.epoch; ++h) {
            if (h < R) {
                const float inv = lt[h] > 0.f ? 1.f / lt[h] : 0.f;
                p.out_o[(orow0 + h) * D + tid] = __uint_as_float(ov[h]) * inv;   // d = tid: coalesced
                if (tid == 0) {
                    const bool any = lt[h] > 0.f;
                    p.out_stats[(orow0 + h) * 2 + 0] = any ? m_run[h] / kLog2e : -INFINITY;
                    p.out_stats[(orow0 + h) * 2 + 1] = any ? lt[h] * ex2(m_use[h] - m_run[h]) : 0.f;
                }
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc<Shape<N>::TMEM_COLS>(tmem);
}

bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);

bool k2_gqa_tc_eligible(const K2Params& p, int d, int qdt, int kvdt) {
    const int64_t G = p.q_heads / p.kv_heads;
    return d == 128 && qdt == SDA_BF16 && kvdt == SDA_BF16 && G > 1 && G * p.q_rows <= 32;
}

template <int N>
static cudaError_t launch_gqa_n(const K2Params& q, cudaStream_t st) {
    using namespace k2g;
    using S = Shape<N>;
    {
        const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k2_gqa_tc_kernel<N>), S::SMEM);
        if (e != cudaSuccess) return e;
    }
    K2GqaParams p;
    p.q_rows = q.q_rows;
    p.kv_cap = q.kv_cap;
    p.kv_len = q.kv_len;
    p.out_o = q.out_o;
    p.out_stats = q.out_stats;
    p.n_batch = q.n_batch;
    p.q_heads = q.q_heads;
    p.kv_heads = q.kv_heads;
    p.n_splits = q.n_splits;
    p.rows = (int)((q.q_heads / q.kv_heads) * q.q_rows);
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
    p.epoch = q.epoch;
    p.b_per = q.b_per;
    for (int i = 0; i < kMaxPeers; ++i) p.ll_rec[i] = q.ll_rec[i];
    CUtensorMap qm, km, vm;
    if (!make_tmap_bf16_2d(&qm, q.q, q.n_batch * q.q_heads * q.q_rows, D, N) ||
        !make_tmap_bf16_2d(&km, q.k, q.n_batch * q.kv_heads * q.kv_cap, D, TILE) ||
        !make_tmap_bf16_2d(&vm, q.v, q.n_batch * q.kv_heads * q.kv_cap, D, TILE))
        return cudaErrorInvalidValue;
    const dim3 grid(1u, (unsigned)q.kv_heads, (unsigned)(q.n_batch * q.n_splits));
    k2_gqa_tc_kernel<N><<<grid, 192, S::SMEM, st>>>(p, qm, km, vm);
    return cudaGetLastError();
}

cudaError_t launch_k2_gqa_tc(const K2Params& q, cudaStream_t st) {
    const int64_t R = (q.q_heads / q.kv_heads) * q.q_rows;
    return R <= 16 ? launch_gqa_n<16>(q, st) : launch_gqa_n<32>(q, st);
}

}  // namespace sda
