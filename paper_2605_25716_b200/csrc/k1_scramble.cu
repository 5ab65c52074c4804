// k1_scramble.cu -- K1: feature scramble (phi / phi^{-T}) fused with the token permutation
// and the single RNE rounding into the cache / wire layout.
//
// Replaces apply_phi / apply_phi_inv_t + permute_rows_gather (scrambler.cpp:42-85,
// permutation.cpp:58-67) as called by enc_qkv (scrambler.cpp:126-136), the inquirer's Q
// scramble (protocol.cpp:885-891) and the context owner's KV shipping
// (protocol.cpp:993-1001).
//
// SIMT design (HBM-bound: 4 B/elem moved vs ~10 flop/elem): every output row is owned by a
// group of LPR = d/16 lanes, 16 elements per lane. P1 is applied as a scatter into shared
// memory, the Walsh-Hadamard butterflies run 4 stages in registers plus log2(LPR) shuffle
// stages, and P2 is applied as a gather from shared memory. Row permutation is a gather on
// the input side (output rows are written in order), so stores stay contiguous.
#include <type_traits>

#include "common.cuh"
#include "quant.cuh"

namespace sda {

template <int D>
struct K1Shape {
    static constexpr int E = D < 16 ? D : 16; // elements per lane (d < 16: one lane owns a row)
    static constexpr int LPR = D / E;         // lanes per row
    static constexpr int R = 32 / LPR;        // rows per warp
    static constexpr int CS = E + 4;          // padded chunk stride (conflict-free LDS/STS.128)
    static constexpr int RS = LPR * CS;       // row stride in smem (floats)
    static constexpr int WARPS = 4;
    static constexpr int ROWS_PER_CTA = 64 > WARPS * R ? 64 : WARPS * R;
    static constexpr int ITERS = ROWS_PER_CTA / (WARPS * R);
};

// E consecutive logical elements starting at `elem` (a multiple of 4) of an LL buffer:
// bf16 -> one u32 of two values per 8 bytes, f32 -> one value per 8 bytes (ll_store).
template <int E, typename T>
__device__ __forceinline__ void ll_store_row(void* base, int64_t elem, const float* v, uint32_t ep) {
    uint8_t* b = static_cast<uint8_t*>(base);
    if constexpr (std::is_same<T, float>::value) {
#pragma unroll
        for (int m = 0; m < E / 2; ++m)
            ll_store(b + 8 * (elem + 2 * m), __float_as_uint(v[2 * m]), __float_as_uint(v[2 * m + 1]), ep);
    } else {
#pragma unroll
        for (int m = 0; m < E / 4; ++m) {
            __nv_bfloat162 x = __floats2bfloat162_rn(v[4 * m], v[4 * m + 1]);
            __nv_bfloat162 y = __floats2bfloat162_rn(v[4 * m + 2], v[4 * m + 3]);
            ll_store(b + 8 * ((elem >> 1) + 2 * m), *reinterpret_cast<uint32_t*>(&x), *reinterpret_cast<uint32_t*>(&y), ep);
        }
    }
}

__device__ __forceinline__ int k1_sidx(int j) { return (j >> 4) * 20 + (j & 15); }

// FLAT (rows == 1, the decode Q): every lane group owns one (request, head) row, so one CTA
// covers WARPS * R rows of the flattened [n_batch][n_heads] space instead of one (b, h) per CTA
// with 63 of its 64 row slots idle.
// QP (the quantised wire, sda_scramble_quant): 0 none; 1 min / max pass -- the scrambled values of
// every (request, head) tensor reduced into p.qscratch, nothing stored; 2 -- the scrambled values
// quantised and dequantised with their tensor's parameters before the one store (wire_round,
// model.cpp:338-341, on the f32 scrambled values)
template <int D, typename Tin, typename Tout, bool FLAT, int QP = 0>
__global__ void __launch_bounds__(128) k1_scramble_kernel(const K1Params p, const int64_t n_batch) {
    using S = K1Shape<D>;
    constexpr int E = S::E, LPR = S::LPR, R = S::R;
    constexpr int ITERS = FLAT ? 1 : S::ITERS;
    __shared__ __align__(16) float sbuf[S::WARPS][R * S::RS];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / LPR, lg = lane % LPR;
    int64_t b;
    int h;
    bool row_ok = true;
    if constexpr (FLAT) {
        int64_t f = (int64_t)blockIdx.x * (S::WARPS * R) + warp * R + g;
        row_ok = f < n_batch * p.n_heads;
        if (!row_ok) f = 0;
        b = f / p.n_heads;
        h = (int)(f % p.n_heads);
    } else {
        h = blockIdx.y;
        b = blockIdx.z;
    }
    const int kh = h / (p.n_heads / p.key_heads);
    const uint8_t* sc = scrambler_ptr(p.keys, p.keys_bstride, b, kh, D, p.which);
    const float* ftab = reinterpret_cast<const float*>(sc);
    const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + 24 * D);

    // This lane's key material for its element chunk [lg*E, lg*E+E).
    float kin[E], kout[E];
    int p1[E], p2i[E];
    {
        const float* fin = ftab + (p.inv_t ? kInInvT : kInFwd) * D + lg * E;
        const float* fout = ftab + (p.inv_t ? kOutInvT : kOutFwd) * D + lg * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            kin[e] = fin[e];
            kout[e] = fout[e];
            p1[e] = k1_sidx(utab[kP1 * D + lg * E + e]);
            p2i[e] = k1_sidx(utab[kP2Inv * D + lg * E + e]);
        }
    }

    const int64_t xb = p.x_batch_mod > 0 ? b % p.x_batch_mod : b;
    const Tin* x = static_cast<const Tin*>(p.x) + (xb * p.n_heads + h) * p.rows * D;
    // LL exchange: write straight into the destination's receive slot, epoch-tagged
    const bool ll = FLAT && p.epoch != nullptr;
    const uint32_t ep = ll ? *p.epoch : 0u;
    pdl_trigger();   // K2 may launch right away (it waits on K1's grid, or spins on the LL words)
    const int64_t out_elem = ((ll ? xb : b) * p.n_heads + h) * p.out_rows_cap * D + p.out_row_offset * D;
    Tout* out = ll ? nullptr : static_cast<Tout*>(p.out) + out_elem;
    const uint32_t* perm = p.perm ? p.perm + b * p.perm_bstride : nullptr;
    float* u = &sbuf[warp][g * S::RS];
    const int64_t qt = b * p.n_heads + h;   // quantisation tensor (request, head)
    const int64_t n_t = n_batch * p.n_heads;
    double qlo = INFINITY, qhi = -INFINITY;
    bool qbad = false;
    QParams qp;
    if constexpr (QP == 2) qp = qparams(p.qscratch, p.qscratch + n_t, qt, p.quant_bits);

    for (int it = 0; it < ITERS; ++it) {
        const int64_t r = FLAT ? 0 : (int64_t)blockIdx.x * S::ROWS_PER_CTA + (int64_t)it * S::WARPS * R + warp * R + g;
        const bool valid = row_ok && r < p.rows;
        const int64_t src = valid ? (perm ? (int64_t)perm[r] : r) : 0;

        float v[E];
        load_vec_n<E>(x + src * D + lg * E, v);
#pragma unroll
        for (int e = 0; e < E; ++e) u[p1[e]] = v[e] * kin[e];   // u[P1[i]] = x[i] * s1^{+-1}[i]
        __syncwarp();
#pragma unroll
        for (int c = 0; c < E / 4; ++c) {
            const float4 t = *reinterpret_cast<const float4*>(&u[lg * S::CS + 4 * c]);
            v[4 * c] = t.x; v[4 * c + 1] = t.y; v[4 * c + 2] = t.z; v[4 * c + 3] = t.w;
        }
        fwht_group<E, LPR>(v, lane);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < E / 4; ++c)
            *reinterpret_cast<float4*>(&u[lg * S::CS + 4 * c]) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = u[p2i[e]] * kout[e];  // y[k] = H(u)[P2inv[k]] * s2^{+-1}[k]/sqrt(d)
        if constexpr (QP == 1) {
            if (valid)
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    qbad |= !isfinite(v[e]);
                    qlo = fmin(qlo, (double)v[e]);
                    qhi = fmax(qhi, (double)v[e]);
                }
            __syncwarp();
            continue;
        }
        if constexpr (QP == 2) {
#pragma unroll
            for (int e = 0; e < E; ++e) v[e] = __double2float_rn(qround((double)v[e], qp));
        }
        if (valid) {
            if (ll)
                ll_store_row<E, Tout>(p.ll_out[b / p.x_batch_mod], out_elem + r * D + lg * E, v, ep);
            else
                store_vec_any<E>(out + r * D + lg * E, v);
        }
        __syncwarp();
    }
    if constexpr (QP == 1) {   // per lane group (FLAT: one tensor per group) or per warp (one tensor per CTA)
        if (qbad && p.qerr) atomicExch(p.qerr, (int32_t)SDA_ERR_INVALID_ARGUMENT);
#pragma unroll
        for (int m = 1; m < (FLAT ? LPR : 32); m <<= 1) {
            qlo = fmin(qlo, __shfl_xor_sync(0xffffffffu, qlo, m));
            qhi = fmax(qhi, __shfl_xor_sync(0xffffffffu, qhi, m));
        }
        if ((FLAT ? lg == 0 : lane == 0) && qlo <= qhi) {
            atomicMin(p.qscratch + qt, dkey(qlo));
            atomicMax(p.qscratch + n_t + qt, dkey(qhi));
        }
    }
}

template <int D, typename Tin, typename Tout, int QP>
static cudaError_t launch_k1_q(const K1Params& p, int64_t n_batch, cudaStream_t st) {
    using S = K1Shape<D>;
    if (p.rows == 1) {
        const int64_t n = n_batch * p.n_heads, per = S::WARPS * S::R;
        k1_scramble_kernel<D, Tin, Tout, true, QP><<<(unsigned)((n + per - 1) / per), 128, 0, st>>>(p, n_batch);
        return cudaGetLastError();
    }
    const dim3 grid((unsigned)((p.rows + S::ROWS_PER_CTA - 1) / S::ROWS_PER_CTA), (unsigned)p.n_heads,
                    (unsigned)n_batch);
    k1_scramble_kernel<D, Tin, Tout, false, QP><<<grid, 128, 0, st>>>(p, n_batch);
    return cudaGetLastError();
}

template <int D, typename Tin, typename Tout>
static cudaError_t launch_k1_t(const K1Params& p, int64_t n_batch, cudaStream_t st) {
    if (p.quant_bits <= 0) return launch_k1_q<D, Tin, Tout, 0>(p, n_batch, st);
    // quantised wire: min / max pass, then the pass that quantises in its epilogue
    const int64_t n_t = n_batch * p.n_heads;
    cudaError_t e = cudaMemsetAsync(p.qscratch, 0xFF, n_t * 8, st);          // min keys
    if (e == cudaSuccess) e = cudaMemsetAsync(p.qscratch + n_t, 0x00, n_t * 8, st);   // max keys
    if (e == cudaSuccess) e = launch_k1_q<D, Tin, Tout, 1>(p, n_batch, st);
    if (e == cudaSuccess) e = launch_k1_q<D, Tin, Tout, 2>(p, n_batch, st);
    return e;
}

template <int D>
static cudaError_t launch_k1_d(const K1Params& p, int xdt, int odt, int64_t n_batch, cudaStream_t st) {
    if (xdt == SDA_BF16 && odt == SDA_BF16) return launch_k1_t<D, __nv_bfloat16, __nv_bfloat16>(p, n_batch, st);
    if (xdt == SDA_BF16 && odt == SDA_F32) return launch_k1_t<D, __nv_bfloat16, float>(p, n_batch, st);
    if (xdt == SDA_F32 && odt == SDA_BF16) return launch_k1_t<D, float, __nv_bfloat16>(p, n_batch, st);
    return launch_k1_t<D, float, float>(p, n_batch, st);
}

cudaError_t launch_k1(const K1Params& p, int d, int xdt, int odt, int64_t n_batch, cudaStream_t st) {
    switch (d) {
        case 4: return launch_k1_d<4>(p, xdt, odt, n_batch, st);
        case 8: return launch_k1_d<8>(p, xdt, odt, n_batch, st);
        case 16: return launch_k1_d<16>(p, xdt, odt, n_batch, st);
        case 32: return launch_k1_d<32>(p, xdt, odt, n_batch, st);
        case 64: return launch_k1_d<64>(p, xdt, odt, n_batch, st);
        case 128: return launch_k1_d<128>(p, xdt, odt, n_batch, st);
        case 256: return launch_k1_d<256>(p, xdt, odt, n_batch, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sda
