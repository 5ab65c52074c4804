// f64_path.cu -- the FP64 mode of K1 / K2 / K3 (x, q, kv and out dtype SDA_F64).
//
// The reference computes the whole path in f64; its exactness gates compare the
// federated result with centralized decoding at 1e-8 (acceptance_main.cpp:50-116,
// test_model.cpp:90-110). This mode runs the same arithmetic on the device in the reference's own
// operation order, every product / quotient / sum explicitly rounded (__dmul_rn, __ddiv_rn,
// __dadd_rn: no FMA contraction), so
//   K1 apply_phi / apply_phi_inv_t + the row gather (scrambler.cpp:42-63)        -- bit-exact,
//   K3 dec_output's apply_phi_inv + scatter (scrambler.cpp:138-149), merge_shards
//      (attention.cpp:89-123)                                                    -- bit-exact up to exp(),
//   K2 shard_attention (attention.cpp:42-78): logits bit-exact, the exp-weighted sums in the
//      reference's key order                                                      -- up to exp(),
// where exp() is CUDA's (<= 1 ulp) against glibc's. Key material comes from the f64 key image
// (sda_pack_keyset_f64: raw s1 / s2, the permutations and their inverses). It is a precision mode
// for oracle-exact runs of the reference's own tests, not a throughput path: one thread per row
// in K1 / K3 (local arrays), one warp per query row in K2.
#include <cmath>

#include "common.cuh"

namespace sda {

__host__ __device__ __forceinline__ const uint8_t* scrambler_ptr_f64(const void* keys, int64_t batch_stride, int64_t b,
                                                                     int kh, int d, int which) {
    return static_cast<const uint8_t*>(keys) + b * batch_stride + (int64_t)kh * SDA_KEYSET_HEAD_BYTES_F64(d) +
           (int64_t)which * SDA_SCRAMBLER_BYTES_F64(d);
}

// fwht_normalized_inplace (fwht.cpp:10-26): butterflies half = 1, 2, ..., then one global scale
template <int D>
__device__ __forceinline__ void fwht_f64(double* x) {
    for (int half = 1; half < D; half <<= 1)
        for (int base = 0; base < D; base += half << 1)
            for (int i = base; i < base + half; ++i) {
                const double a = x[i], b = x[i + half];
                x[i] = __dadd_rn(a, b);
                x[i + half] = __dsub_rn(a, b);
            }
    const double scale = 1.0 / sqrt((double)D);
    for (int i = 0; i < D; ++i) x[i] = __dmul_rn(x[i], scale);
}

// apply_row (scrambler.cpp:42-63) for one row: variant 0 forward, 1 inv_t, 2 inv
template <int D>
__device__ __forceinline__ void apply_row_f64(const double* in, double* out, const uint8_t* sc, int variant) {
    const double* s1 = reinterpret_cast<const double*>(sc);
    const double* s2 = s1 + D;
    const uint16_t* u = reinterpret_cast<const uint16_t*>(sc + 16 * D);
    const uint16_t* P1 = u + kP1 * D;
    const uint16_t* P2 = u + kP2 * D;
    double tmp[D], o[D];
    if (variant == 2) {   // x S2^-1 P2^T H P1^T S1^-1
        for (int i = 0; i < D; ++i) tmp[i] = __ddiv_rn(in[i], s2[i]);
        for (int i = 0; i < D; ++i) o[i] = tmp[P2[i]];   // permute_gather
        fwht_f64<D>(o);
        for (int i = 0; i < D; ++i) tmp[i] = o[P1[i]];
        for (int i = 0; i < D; ++i) out[i] = __ddiv_rn(tmp[i], s1[i]);
        return;
    }
    const bool inv = variant == 1;
    for (int i = 0; i < D; ++i) tmp[i] = inv ? __ddiv_rn(in[i], s1[i]) : __dmul_rn(in[i], s1[i]);
    for (int i = 0; i < D; ++i) o[P1[i]] = tmp[i];      // permute_scatter
    fwht_f64<D>(o);
    for (int i = 0; i < D; ++i) tmp[P2[i]] = o[i];
    for (int i = 0; i < D; ++i) out[i] = inv ? __ddiv_rn(tmp[i], s2[i]) : __dmul_rn(tmp[i], s2[i]);
}

// K1: out[b][h][off + r] = apply(x[b'][h][perm_b[r]]), one thread per output row
template <int D>
__global__ void __launch_bounds__(128) k1_f64_kernel(const K1Params p) {
    const int h = blockIdx.y;
    const int64_t b = blockIdx.z;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= p.rows) return;
    const int kh = h / (p.n_heads / p.key_heads);
    const uint8_t* sc = scrambler_ptr_f64(p.keys, p.keys_bstride, b, kh, D, p.which);
    const int64_t xb = p.x_batch_mod > 0 ? b % p.x_batch_mod : b;
    const int64_t src = p.perm ? (int64_t)p.perm[b * p.perm_bstride + r] : r;   // permute_rows_gather
    const double* x = static_cast<const double*>(p.x) + ((xb * p.n_heads + h) * p.rows + src) * D;
    double* out = static_cast<double*>(p.out) + ((b * p.n_heads + h) * p.out_rows_cap + p.out_row_offset + r) * D;
    double in[D], y[D];
    for (int i = 0; i < D; ++i) in[i] = x[i];
    apply_row_f64<D>(in, y, sc, p.inv_t ? 1 : 0);
    for (int i = 0; i < D; ++i) out[i] = y[i];
}

// K2: shard_attention for one (split, q head, request x q row), one warp. Logits of 32 keys at a
// time (lane j: dot(q, k_j) summed over c in order, times the scale); pass 1 takes the max, pass 2
// recomputes them (identical values), exponentiates, and every lane adds w_j v_j to the output
// columns it owns in key order -- the reference's exact summation order.
template <int D>
__global__ void __launch_bounds__(32) k2_f64_kernel(const K2Params p) {
    __shared__ double qs[D];
    const int lane = threadIdx.x;
    const int split = blockIdx.x, h = blockIdx.y;
    const int64_t b = (int64_t)blockIdx.z / p.q_rows, qr = (int64_t)blockIdx.z % p.q_rows;
    const int kvh = h / (p.q_heads / p.kv_heads);
    int64_t len = p.kv_len ? (int64_t)p.kv_len[b] : p.kv_cap;
    if (p.causal) {
        const int64_t lim = qr + p.causal_offset + 1;
        len = lim < 0 ? 0 : (lim < len ? lim : len);
    }
    const int64_t tiles = (len + 127) / 128;
    const int64_t chunk = ((tiles + p.n_splits - 1) / p.n_splits) * 128;
    const int64_t k0 = (int64_t)split * chunk, k1 = min(len, k0 + chunk);
    const double* q = static_cast<const double*>(p.q) + ((b * p.q_heads + h) * p.q_rows + qr) * D;
    for (int c = lane; c < D; c += 32) qs[c] = q[c];
    __syncwarp();
    const double* kb = static_cast<const double*>(p.k) + (b * p.kv_heads + kvh) * p.kv_cap * D;
    const double* vb = static_cast<const double*>(p.v) + (b * p.kv_heads + kvh) * p.kv_cap * D;
    const double scale = 1.0 / sqrt((double)D);   // attention.cpp:45
    auto logit = [&](int64_t j) {
        const double* kr = kb + j * D;
        double s = 0.0;
        for (int c = 0; c < D; ++c) s = __dadd_rn(s, __dmul_rn(qs[c], kr[c]));   // dot (matrix.cpp:89-93)
        return __dmul_rn(s, scale);
    };
    double m = -INFINITY;
    for (int64_t j0 = k0; j0 < k1; j0 += 32) {
        const int64_t j = j0 + lane;
        if (j < k1) m = fmax(m, logit(j));
    }
    for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    constexpr int E = (D + 31) / 32;
    double acc[E];
    for (int e = 0; e < E; ++e) acc[e] = 0.0;
    double s = 0.0;
    if (m > -INFINITY) {
        for (int64_t j0 = k0; j0 < k1; j0 += 32) {
            const int64_t j = j0 + lane;
            const double w_l = j < k1 ? exp(__dsub_rn(logit(j), m)) : 0.0;
            const int n = (int)(k1 - j0 < 32 ? k1 - j0 : 32);
            for (int t = 0; t < n; ++t) {
                const double w = __shfl_sync(0xffffffffu, w_l, t);
                s = __dadd_rn(s, w);
                const double* vr = vb + (j0 + t) * D;
                for (int e = 0; e < E; ++e) {
                    const int c = lane + 32 * e;
                    if (c < D) acc[e] = __dadd_rn(acc[e], __dmul_rn(w, vr[c]));
                }
            }
        }
    }
    const int64_t orow = ((int64_t)split * p.n_batch * p.q_heads + b * p.q_heads + h) * p.q_rows + qr;
    double* oo = reinterpret_cast<double*>(p.out_o) + orow * D;
    for (int e = 0; e < E; ++e) {
        const int c = lane + 32 * e;
        if (c < D) oo[c] = s > 0.0 ? __ddiv_rn(acc[e], s) : 0.0;
    }
    if (lane == 0) {
        double* st = reinterpret_cast<double*>(p.out_stats) + orow * 2;
        st[0] = s > 0.0 ? m : -INFINITY;   // fully masked: exp_sum 0 (attention.cpp:66-67)
        st[1] = s;
    }
}

// K3: per output row, every keyed source unscrambled on its own (dec_output: apply_phi_inv of
// O' row p_q^-1[r], stats of the same row) and then merge_shards over the sources in order; one
// source is returned verbatim. One thread per row.
template <int D>
__global__ void __launch_bounds__(128) k3_f64_kernel(const K3Params p) {
    const int64_t total = p.n_batch * p.q_heads * p.q_rows;
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= total) return;
    const int64_t r = row % p.q_rows, bh = row / p.q_rows;
    const int h = (int)(bh % p.q_heads);
    const int64_t b = bh / p.q_heads;
    const int kh = h / (p.q_heads / p.key_heads);
    auto offs = [&](const K3Source& src, int64_t& st_off, int64_t& o_off) {
        const int64_t ri = src.pq_inv ? (int64_t)src.pq_inv[b * p.pq_bstride + r] : r;
        st_off = src.bstride ? b * src.bstride + ((int64_t)h * p.q_rows + ri) * 2 : (bh * p.q_rows + ri) * 2;
        o_off = src.bstride ? b * src.bstride + ((int64_t)h * p.q_rows + ri) * D : (bh * p.q_rows + ri) * D;
    };
    auto stats = [&](int s) {
        int64_t so, oo;
        offs(p.src[s], so, oo);
        const double* st = reinterpret_cast<const double*>(p.src[s].stats) + so;
        return make_double2(st[0], st[1]);
    };
    auto load_row = [&](int s, double* y) {
        int64_t so, oo;
        offs(p.src[s], so, oo);
        const double* o = reinterpret_cast<const double*>(p.src[s].o) + oo;
        if (p.src[s].keys) {
            double in[D];
            for (int i = 0; i < D; ++i) in[i] = o[i];
            apply_row_f64<D>(in, y, scrambler_ptr_f64(p.src[s].keys, p.keys_bstride, b, kh, D, 1), 2);
        } else {
            for (int i = 0; i < D; ++i) y[i] = o[i];
        }
    };
    double out[D];
    double2 res_st;
    bool masked;
    if (p.n_src == 1) {   // attention.cpp:97-101 (dec_output alone: the scattered stats as they are)
        res_st = stats(0);
        masked = res_st.y == 0.0;
        load_row(0, out);
    } else {
        double mstar = -INFINITY;
        for (int s = 0; s < p.n_src; ++s) {
            const double2 st = stats(s);
            if (st.y > 0.0 && st.x > mstar) mstar = st.x;
        }
        masked = !(mstar > -INFINITY);
        double denom = 0.0;
        for (int i = 0; i < D; ++i) out[i] = 0.0;
        if (!masked) {
            for (int s = 0; s < p.n_src; ++s) {
                const double2 st = stats(s);
                if (st.y == 0.0) continue;
                const double w = __dmul_rn(st.y, exp(__dsub_rn(st.x, mstar)));
                denom = __dadd_rn(denom, w);
                double y[D];
                load_row(s, y);
                for (int i = 0; i < D; ++i) out[i] = __dadd_rn(out[i], __dmul_rn(w, y[i]));
            }
            for (int i = 0; i < D; ++i) out[i] = __ddiv_rn(out[i], denom);
        }
        res_st = make_double2(mstar, masked ? 0.0 : denom);
    }
    if (masked && p.err) atomicExch(p.err, (int32_t)SDA_ERR_MASKED_ROW);
    const int64_t hr = (int64_t)h * p.q_rows + r;
    double* o = static_cast<double*>(p.out) + (p.out_bstride ? b * p.out_bstride + hr * D : row * D);
    for (int i = 0; i < D; ++i) o[i] = masked && p.n_src > 1 ? NAN : out[i];
    if (p.out_stats) {
        double* so = reinterpret_cast<double*>(p.out_stats) + (p.out_bstride ? b * p.out_bstride + hr * 2 : row * 2);
        so[0] = res_st.x;
        so[1] = res_st.y;
    }
}

template <int D>
static cudaError_t launch_f64(int which, const void* params, int64_t n_batch, cudaStream_t st) {
    if (which == 1) {
        const K1Params& p = *static_cast<const K1Params*>(params);
        k1_f64_kernel<D><<<dim3((unsigned)((p.rows + 127) / 128), (unsigned)p.n_heads, (unsigned)n_batch), 128, 0, st>>>(p);
    } else if (which == 2) {
        const K2Params& p = *static_cast<const K2Params*>(params);
        k2_f64_kernel<D><<<dim3((unsigned)p.n_splits, (unsigned)p.q_heads, (unsigned)(p.n_batch * p.q_rows)), 32, 0, st>>>(p);
    } else {
        const K3Params& p = *static_cast<const K3Params*>(params);
        const int64_t total = p.n_batch * p.q_heads * p.q_rows;
        k3_f64_kernel<D><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(p);
    }
    return cudaGetLastError();
}

// which: 1 K1, 2 K2, 3 K3; params: the K1Params / K2Params / K3Params of the call
cudaError_t launch_f64_path(int which, const void* params, int d, int64_t n_batch, cudaStream_t st) {
    switch (d) {
        case 4: return launch_f64<4>(which, params, n_batch, st);
        case 8: return launch_f64<8>(which, params, n_batch, st);
        case 16: return launch_f64<16>(which, params, n_batch, st);
        case 32: return launch_f64<32>(which, params, n_batch, st);
        case 64: return launch_f64<64>(which, params, n_batch, st);
        case 128: return launch_f64<128>(which, params, n_batch, st);
        case 256: return launch_f64<256>(which, params, n_batch, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sda
