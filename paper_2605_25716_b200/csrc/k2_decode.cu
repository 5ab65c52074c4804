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
#include <algorithm>
#include <cmath>
#include <type_traits>

#include "common.cuh"

namespace sda {

template <int D>
struct K2Shape {
    static constexpr int VEC = D < 8 ? D : 8;    // elements per lane (d = 4: one lane per key row)
    static constexpr int LPR = D / VEC;          // lanes per key row
    static constexpr int RW = 32 / LPR;          // key rows per warp step
    static constexpr int WARPS = 4;
    static constexpr int NG = WARPS * RW;        // lane groups per CTA
    // keys in flight per lane group: 4 keeps the kernel at 56 registers (9 CTAs = 36 warps per
    // SM) -- measured 3-5 % faster on C2 than 8 (86 registers, 5 CTAs per SM) once the split
    // count fills whole waves (sda_default_splits); 2 starves the memory pipe
    static constexpr int U = 4;
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
    const bool ll = p.epoch != nullptr;   // LL exchange (decode): Q' in, the split's record out
    const uint32_t ep = ll ? *p.epoch : 0u;
    if (!ll) pdl_wait();   // launched early behind K1 (PDL): its Q' must be complete; LL spins instead
    pdl_trigger();         // K3 may launch once every K2 CTA is running (it waits on this grid or on LL)

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
    const int64_t q_elem = ((b * p.q_heads + h) * p.q_rows + qr) * D + lg * VEC;
    if (ll) {   // spin until this request's Q' has arrived from its inquirer
        const uint8_t* qb = static_cast<const uint8_t*>(p.q);
        if constexpr (std::is_same<TQ, float>::value) {
#pragma unroll
            for (int m = 0; m < VEC / 2; ++m) {
                const uint2 w = ll_load(qb + 8 * (q_elem + 2 * m), ep);
                qv[2 * m] = __uint_as_float(w.x);
                qv[2 * m + 1] = __uint_as_float(w.y);
            }
        } else {
#pragma unroll
            for (int m = 0; m < VEC / 4; ++m) {
                const uint2 w = ll_load(qb + 8 * ((q_elem >> 1) + 2 * m), ep);
                qv[4 * m] = __uint_as_float(w.x << 16);
                qv[4 * m + 1] = __uint_as_float(w.x & 0xFFFF0000u);
                qv[4 * m + 2] = __uint_as_float(w.y << 16);
                qv[4 * m + 3] = __uint_as_float(w.y & 0xFFFF0000u);
            }
        }
    } else {
        load_vec_n<VEC>(static_cast<const TQ*>(p.q) + q_elem, qv);
    }
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
        using Raw = typename std::conditional<VEC == 8, Raw8<TKV>, Raw4<TKV>>::type;
        Raw kr[U], vr[U];
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
    // lane-group weights: in registers up to 32 groups (d >= 32); the small head dims (64 / 128
    // groups) keep them in shared memory instead of spilling a 128-entry array
    constexpr bool WREG = NG <= 32;
    float wgt[WREG ? NG : 1];
    __shared__ float sm_w[WREG ? 1 : NG];
    if constexpr (WREG) {
#pragma unroll
        for (int i = 0; i < NG; ++i) {
            wgt[i] = (M == -INFINITY) ? 0.f : ex2(sm_m[i] - M);
            S_ = fmaf(sm_s[i], wgt[i], S_);
        }
    } else {
        for (int i = threadIdx.x; i < NG; i += blockDim.x) sm_w[i] = (M == -INFINITY) ? 0.f : ex2(sm_m[i] - M);
        __syncthreads();
        for (int i = 0; i < NG; ++i) S_ = fmaf(sm_s[i], sm_w[i], S_);
    }
    auto weight = [&](int i) -> float {
        if constexpr (WREG) return wgt[i];
        else return sm_w[i];
    };
    const float inv = S_ > 0.f ? 1.f / S_ : 0.f;
    // back to natural-log units: row_max = max_j q.k_j / sqrt(d)
    const float row_max = S_ > 0.f ? M / kLog2e : -INFINITY;
    if (ll) {   // the split's record row, straight into the inquirer's receive slot
        const int64_t dest = b / p.b_per, i = b % p.b_per;
        uint8_t* rb = static_cast<uint8_t*>(p.ll_rec[dest]) + 8 * (((split * p.b_per + i) * p.q_heads + h) * (D + 2));
        for (int pr = threadIdx.x; pr < D / 2; pr += blockDim.x) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int g2 = 0; g2 < NG; ++g2) {
                a0 = fmaf(sm_o[g2][2 * pr], weight(g2), a0);
                a1 = fmaf(sm_o[g2][2 * pr + 1], weight(g2), a1);
            }
            ll_store(rb + 16 * pr, __float_as_uint(a0 * inv), __float_as_uint(a1 * inv), ep);
        }
        if (threadIdx.x == 0) ll_store(rb + 8 * D, __float_as_uint(row_max), __float_as_uint(S_), ep);
        pdl_wait();   // K2 completes only after K1 has (stream order for the next step)
        return;
    }
    const int64_t orow = ((int64_t)split * p.n_batch * p.q_heads + b * p.q_heads + h) * p.q_rows + qr;
    for (int dim = threadIdx.x; dim < D; dim += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < NG; ++i) acc = fmaf(sm_o[i][dim], weight(i), acc);
        p.out_o[orow * D + dim] = acc * inv;
    }
    if (threadIdx.x == 0) {
        p.out_stats[orow * 2 + 0] = row_max;
        p.out_stats[orow * 2 + 1] = S_;
    }
}

template <int D, typename TQ, typename TKV>
static cudaError_t launch_k2_t(const K2Params& p, cudaStream_t st) {
    const dim3 grid((unsigned)p.n_splits, (unsigned)p.q_heads, (unsigned)(p.n_batch * p.q_rows));
    return pdl_launch(k2_decode_kernel<D, TQ, TKV>, grid, dim3(128), st, p);
}

template <int D>
static cudaError_t launch_k2_d(const K2Params& p, int qdt, int kvdt, cudaStream_t st) {
    if (qdt == SDA_BF16 && kvdt == SDA_BF16) return launch_k2_t<D, __nv_bfloat16, __nv_bfloat16>(p, st);
    if (qdt == SDA_F32 && kvdt == SDA_BF16) return launch_k2_t<D, float, __nv_bfloat16>(p, st);
    if (qdt == SDA_BF16 && kvdt == SDA_F32) return launch_k2_t<D, __nv_bfloat16, float>(p, st);
    return launch_k2_t<D, float, float>(p, st);
}

// LL Q' (bf16 wire: 4 values per 16-byte word) -> plain bf16 rows for the TMA-fed tensor-core
// GQA kernel; spins until the words carry the step's epoch
__global__ void __launch_bounds__(256) ll_unpack_q_kernel(const uint8_t* __restrict__ ll, int64_t words, uint2* out,
                                                          const uint32_t* epoch) {
    const uint32_t ep = *epoch;
    pdl_trigger();
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
        out[w] = ll_load(ll + 16 * w, ep);
}

cudaError_t launch_ll_unpack_q(const void* ll_q, int64_t elems, void* out, const uint32_t* epoch, cudaStream_t st) {
    const int64_t words = elems / 4;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((words + 255) / 256, 1184));
    return pdl_launch(ll_unpack_q_kernel, dim3(blocks), dim3(256), st, static_cast<const uint8_t*>(ll_q), words,
                      static_cast<uint2*>(out), epoch);
}

SDA_SPIN_ACCESSOR(spin_access_k2_decode)

int k2_decode_ctas_per_sm() {   // resident CTAs per SM of the C2 instantiation (split heuristic)
    static int n = 0;
    if (!n) {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k2_decode_kernel<128, __nv_bfloat16, __nv_bfloat16>, 128, 0) !=
                cudaSuccess ||
            b <= 0) {
            cudaGetLastError();
            b = 9;   // no device (CPU-side callers): the sm_100a build's value (56 registers)
        }
        n = b;
    }
    return n;
}

cudaError_t launch_k2_decode(const K2Params& p, int d, int qdt, int kvdt, cudaStream_t st) {
    switch (d) {
        case 4: return launch_k2_d<4>(p, qdt, kvdt, st);
        case 8: return launch_k2_d<8>(p, qdt, kvdt, st);
        case 16: return launch_k2_d<16>(p, qdt, kvdt, st);
        case 32: return launch_k2_d<32>(p, qdt, kvdt, st);
        case 64: return launch_k2_d<64>(p, qdt, kvdt, st);
        case 128: return launch_k2_d<128>(p, qdt, kvdt, st);
        case 256: return launch_k2_d<256>(p, qdt, kvdt, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sda
