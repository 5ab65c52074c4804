// k2_decode.cu -- K2 (decode / few-row form): keyless split-KV partial attention.
//
// Replaces shard_attention(q', K', V', none) (attention.cpp:42-78) as the compute node runs
// it in try_serve_q (protocol.cpp:1072-1095) -- without the per-call concatenation copy of
// the domain's segments (:1073-1085): the KV shard stays resident as one [kv_cap x d] slab
// per (request, kv head) and the kernel reads it in place.
//
// Decode is purely HBM-bound (each request owns its own key set, so scrambled KV is never
// shared: ~1 flop/B for MHA). Design: one CTA per (split, q head, request x q row); 16-byte
// streaming loads (8 elements per lane, d/8 lanes per key row, U keys in flight per lane);
// warp-shuffle dot-product reduction; per-lane-group online softmax in f32; a final
// shared-memory merge of the CTA's lane groups. Emits the split's locally normalised O'
// and (row_max, exp_sum) exactly as ShardStats defines them (attention.hpp:34-41).
#include <cmath>

#include "common.cuh"

namespace sda {

template <int D>
struct K2Shape {
    static constexpr int VEC = 8;
    static constexpr int LPR = D / VEC;          // lanes per key row
    static constexpr int RW = 32 / LPR;          // key rows per warp step
    static constexpr int WARPS = 4;
    static constexpr int NG = WARPS * RW;        // lane groups per CTA
    static constexpr int U = 8;                  // keys in flight per lane group
};

template <int D, typename TQ, typename TKV>
__global__ void __launch_bounds__(128) k2_decode_kernel(const K2Params p) {
    using S = K2Shape<D>;
    constexpr int VEC = S::VEC, LPR = S::LPR, NG = S::NG, U = S::U;
    __shared__ float sm_m[NG], sm_s[NG];
    __shared__ __align__(16) float sm_o[NG][D];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / LPR, lg = lane % LPR;
    const int grp = warp * S::RW + g;
    const int split = blockIdx.x, h = blockIdx.y;
    const int64_t b = (int64_t)blockIdx.z / p.q_rows, qr = (int64_t)blockIdx.z % p.q_rows;
    const int kvh = h / (p.q_heads / p.kv_heads);
    if (p.wait_flags) {   // fused exchange: this request's Q' must have arrived from its inquirer
        if (threadIdx.x == 0) flag_wait(p.wait_flags + b / p.wait_group, *p.epoch);
        __syncthreads();
    }

    int64_t len = p.kv_len ? (int64_t)p.kv_len[b] : p.kv_cap;
    if (p.causal) {   // keys j <= qr + offset only (AttentionMask::causal, attention.cpp:16-27)
        const int64_t lim = qr + p.causal_offset + 1;
        len = lim < 0 ? 0 : (lim < len ? lim : len);
    }
    // splits are whole 128-key tiles (the same ranges as the tensor-core kernels)
    const int64_t tiles = (len + 127) / 128;
    const int64_t chunk = ((tiles + p.n_splits - 1) / p.n_splits) * 128;
    const int64_t k0 = (int64_t)split * chunk;
    const int64_t k1 = min(len, k0 + chunk);

    float qv[VEC];
    load_vec<VEC>(static_cast<const TQ*>(p.q) + ((b * p.q_heads + h) * p.q_rows + qr) * D + lg * VEC, qv);
#pragma unroll
    for (int i = 0; i < VEC; ++i) qv[i] *= p.scale * kLog2e;   // logits in log2 units

    const TKV* kb = static_cast<const TKV*>(p.k) + ((b * p.kv_heads + kvh) * p.kv_cap) * D + lg * VEC;
    const TKV* vb = static_cast<const TKV*>(p.v) + ((b * p.kv_heads + kvh) * p.kv_cap) * D + lg * VEC;

    float m = -INFINITY, s = 0.f;
    float o[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) o[i] = 0.f;

    // The loop bound is warp-uniform (every lane of the warp runs the same trip count) so the
    // full-mask shuffles below are always executed by all 32 lanes; rows past k1 are masked.
    for (int64_t jw = k0 + warp * S::RW; jw < k1; jw += (int64_t)NG * U) {
        const int64_t j0 = jw + g;
        Raw8<TKV> kr[U], vr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = j0 + (int64_t)u * NG;
            const int64_t jj = j < k1 ? j : k0;
            kr[u].load(kb + jj * D);
            vr[u].load(vb + jj * D);
        }
        float l[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc = fmaf(qv[i], kr[u].get(i), acc);
#pragma unroll
            for (int msk = LPR / 2; msk >= 1; msk >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, msk);
            l[u] = (j0 + (int64_t)u * NG < k1) ? acc : -INFINITY;
        }
        float mn = m;
#pragma unroll
        for (int u = 0; u < U; ++u) mn = fmaxf(mn, l[u]);
        if (mn == -INFINITY) continue;     // this lane group has no valid row yet (ragged tail)
        const float alpha = ex2(m - mn);   // m = -inf -> 0
        s *= alpha;
#pragma unroll
        for (int i = 0; i < VEC; ++i) o[i] *= alpha;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float pu = ex2(l[u] - mn);
            s += pu;
#pragma unroll
            for (int i = 0; i < VEC; ++i) o[i] = fmaf(pu, vr[u].get(i), o[i]);
        }
        m = mn;
    }

    if (lg == 0) {
        sm_m[grp] = m;
        sm_s[grp] = s;
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i) sm_o[grp][lg * VEC + i] = o[i];
    __syncthreads();

    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < NG; ++i) M = fmaxf(M, sm_m[i]);
    float S_ = 0.f;
    float wgt[NG];
#pragma unroll
    for (int i = 0; i < NG; ++i) {
        wgt[i] = (M == -INFINITY) ? 0.f : ex2(sm_m[i] - M);
        S_ = fmaf(sm_s[i], wgt[i], S_);
    }
    const int64_t orow = ((int64_t)split * p.n_batch * p.q_heads + b * p.q_heads + h) * p.q_rows + qr;
    const float inv = S_ > 0.f ? 1.f / S_ : 0.f;
    for (int dim = threadIdx.x; dim < D; dim += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < NG; ++i) acc = fmaf(sm_o[i][dim], wgt[i], acc);
        p.out_o[orow * D + dim] = acc * inv;
    }
    if (threadIdx.x == 0) {
        // back to natural-log units: row_max = max_j q.k_j / sqrt(d)
        p.out_stats[orow * 2 + 0] = S_ > 0.f ? M / kLog2e : -INFINITY;
        p.out_stats[orow * 2 + 1] = S_;
    }
    if (!p.fold_counters) return;

    // ---- fused exchange: the last split CTA of this row folds the splits (merge_shards in
    // scrambled space, attention.cpp:89-123) and pushes the packed (O', stats) record to the
    // inquirer; the last row of a destination raises its SCR_SHARD flag
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    const int64_t row = (b * p.q_heads + h) * p.q_rows + qr;
    if (threadIdx.x == 0) last = atomicAdd(&p.fold_counters[row], 1u) == (unsigned)p.n_splits - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int64_t split_stride = p.n_batch * p.q_heads * p.q_rows;
    float ms = -INFINITY;
    for (int sp = 0; sp < p.n_splits; ++sp) {
        const float2 st = __ldcg(reinterpret_cast<const float2*>(p.out_stats) + sp * split_stride + row);
        if (st.y > 0.f) ms = fmaxf(ms, st.x);
    }
    float den = 0.f;
    const int64_t dest = b / p.wait_group, i = b % p.wait_group;
    float* rec = p.rec_peer[dest] + i * p.rec_stride;
    const int64_t hr = (int64_t)h * p.q_rows + qr;
    for (int dim = threadIdx.x; dim < D; dim += blockDim.x) {
        float acc = 0.f, dd = 0.f;
        for (int sp = 0; sp < p.n_splits; ++sp) {
            const float2 st = __ldcg(reinterpret_cast<const float2*>(p.out_stats) + sp * split_stride + row);
            if (st.y > 0.f) {
                const float w = st.y * expf(st.x - ms);
                dd += w;
                acc = fmaf(w, __ldcg(p.out_o + (sp * split_stride + row) * D + dim), acc);
            }
        }
        rec[hr * D + dim] = dd > 0.f ? acc / dd : 0.f;
        den = dd;
    }
    if (threadIdx.x == 0) {
        float* st = rec + (int64_t)p.q_heads * p.q_rows * D + hr * 2;
        st[0] = den > 0.f ? ms : -INFINITY;
        st[1] = den;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        p.fold_counters[row] = 0;
        const unsigned rows_per_dest = (unsigned)(p.wait_group * p.q_heads * p.q_rows);
        if (atomicAdd(&p.dest_counters[dest], 1u) == rows_per_dest - 1) {
            p.dest_counters[dest] = 0;
            __threadfence_system();
            flag_raise(p.rec_flag[dest], *p.epoch);
        }
    }
}

template <int D, typename TQ, typename TKV>
static cudaError_t launch_k2_t(const K2Params& p, cudaStream_t st) {
    const dim3 grid((unsigned)p.n_splits, (unsigned)p.q_heads, (unsigned)(p.n_batch * p.q_rows));
    k2_decode_kernel<D, TQ, TKV><<<grid, 128, 0, st>>>(p);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_k2_d(const K2Params& p, int qdt, int kvdt, cudaStream_t st) {
    if (qdt == SDA_BF16 && kvdt == SDA_BF16) return launch_k2_t<D, __nv_bfloat16, __nv_bfloat16>(p, st);
    if (qdt == SDA_F32 && kvdt == SDA_BF16) return launch_k2_t<D, float, __nv_bfloat16>(p, st);
    if (qdt == SDA_BF16 && kvdt == SDA_F32) return launch_k2_t<D, __nv_bfloat16, float>(p, st);
    return launch_k2_t<D, float, float>(p, st);
}

cudaError_t launch_k2_decode(const K2Params& p, int d, int qdt, int kvdt, cudaStream_t st) {
    switch (d) {
        case 32: return launch_k2_d<32>(p, qdt, kvdt, st);
        case 64: return launch_k2_d<64>(p, qdt, kvdt, st);
        case 128: return launch_k2_d<128>(p, qdt, kvdt, st);
        case 256: return launch_k2_d<256>(p, qdt, kvdt, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sda
