// k3_merge.cu -- K3: cross-node LSE-weighted merge + inverse token permutation + unscramble.
//
// Replaces, per output row, dec_output for every remote domain (scrambler.cpp:138-149:
// O = scatter_rows(O' phi_V^{-1}, p_q), stats scattered by p_q) followed by merge_shards
// (attention.cpp:89-123: M* = max row_max over shards with exp_sum > 0,
// w_i = exp_sum_i exp(row_max_i - M*), O = sum w_i O_i / sum w_i), as span_finish_layer
// composes them (protocol.cpp:926-948).
//
// One warp per output row (b, h, r). The scatter by p_q becomes a gather by p_q^{-1} on the
// read side. Because phi_V^{-1} is linear, the weighted sum of every source that shares a
// key set (the K2 splits of one domain) is accumulated in scrambled space and unscrambled
// once per domain: one 128-point FWHT per (row, domain) instead of per split.
// HBM-bound: reads (4d + 8) B per (row, source), writes d * sizeof(out) B per row.
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "quant.cuh"

namespace sda {

// Per-lane slice of one source's phi_V^{-1} tables (and its O' row and stats), loaded one
// source ahead of its use so the dependent HBM / NVLink-written reads of consecutive sources
// overlap instead of forming one latency chain per source.
template <int E>
struct SrcLd {
    float2 st;
    float ov[E];
    float inv_in[E], inv_out[E];
    int p2[E], p1[E];
};

template <int D>
__device__ __forceinline__ void unscramble_acc(const SrcLd<D / 32>& L, float* acc, float* out, float* sh, int lane) {
    constexpr int E = D / 32;
    // t[i] = acc[i] / s2[i] ; u[j] = t[P2[j]] ; w = H u ; y[i] = w[P1[i]] / (s1[i] sqrt(d))
#pragma unroll
    for (int e = 0; e < E; ++e) sh[lane * E + e] = acc[e] * L.inv_in[e];
    __syncwarp();
    float v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = sh[L.p2[e]];
    fwht_group<E, 32>(v, lane);
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) sh[lane * E + e] = v[e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] += sh[L.p1[e]] * L.inv_out[e];
    __syncwarp();
}

template <int D, typename TOut>
__global__ void __launch_bounds__(128) k3_merge_kernel(const K3Params p) {
    constexpr int E = D / 32;
    __shared__ __align__(16) float sh_all[4][D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* sh = sh_all[warp];
    const int64_t total = p.n_batch * p.q_heads * p.q_rows;
    const bool ll = p.ll != 0;   // LL exchange: records arrive epoch-tagged in peer memory
    const uint32_t ep = ll ? *p.epoch : 0u;
    if (!ll) pdl_wait();         // launched early behind K2 (PDL): its partials must be complete
    const int64_t row_raw = (int64_t)blockIdx.x * 4 + warp;
    const bool active = row_raw < total;
    const int64_t row = active ? row_raw : total - 1;   // inactive warps compute a dummy row, store nothing
    const int64_t r = row % p.q_rows;
    const int64_t bh = row / p.q_rows;
    const int h = (int)(bh % p.q_heads);
    const int64_t b = bh / p.q_heads;
    const int kh = h / (p.q_heads / p.key_heads);

    auto offsets = [&](const K3Source& src, int64_t& st_off, int64_t& o_off) {
        if (ll) {   // logical floats of the record row (b, h): [d O' | row_max, exp_sum]
            o_off = b * src.bstride + (int64_t)h * (D + 2);
            st_off = o_off + D;
            return;
        }
        const int64_t ri = src.pq_inv ? (int64_t)src.pq_inv[b * p.pq_bstride + r] : r;
        st_off = src.bstride ? b * src.bstride + ((int64_t)h * p.q_rows + ri) * 2 : (bh * p.q_rows + ri) * 2;
        o_off = src.bstride ? b * src.bstride + ((int64_t)h * p.q_rows + ri) * D : (bh * p.q_rows + ri) * D;
    };

    // pass 1: M* over sources with exp_sum > 0 (attention.cpp:103-105); lanes stride sources,
    // lane s keeps source s's stats for pass 2 (n_src <= 32)
    float mstar = -INFINITY;
    float2 st_lane = make_float2(-INFINITY, 0.f);
    for (int s = lane; s < p.n_src; s += 32) {
        int64_t st_off, o_off;
        offsets(p.src[s], st_off, o_off);
        float2 st;
        if (ll) {
            const uint2 w = ll_load(reinterpret_cast<const uint8_t*>(p.src[s].o) + 8 * st_off, ep);
            st = make_float2(__uint_as_float(w.x), __uint_as_float(w.y));
        } else {
            st = *reinterpret_cast<const float2*>(p.src[s].stats + st_off);
        }
        if (s == lane) st_lane = st;
        if (st.y > 0.f) mstar = fmaxf(mstar, st.x);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) mstar = fmaxf(mstar, __shfl_xor_sync(0xffffffffu, mstar, m));

    auto load_src = [&](int s, SrcLd<E>& L) {
        const K3Source& src = p.src[s];
        int64_t st_off, o_off;
        offsets(src, st_off, o_off);
        const float sx = __shfl_sync(0xffffffffu, st_lane.x, s & 31);
        const float sy = __shfl_sync(0xffffffffu, st_lane.y, s & 31);
        if (ll) {
            const uint8_t* rb = reinterpret_cast<const uint8_t*>(src.o);
            if (p.n_src <= 32) {
                L.st = make_float2(sx, sy);
            } else {
                const uint2 w = ll_load(rb + 8 * st_off, ep);
                L.st = make_float2(__uint_as_float(w.x), __uint_as_float(w.y));
            }
#pragma unroll
            for (int m = 0; m < E / 2; ++m) {
                const uint2 w = ll_load(rb + 8 * (o_off + lane * E + 2 * m), ep);
                L.ov[2 * m] = __uint_as_float(w.x);
                L.ov[2 * m + 1] = __uint_as_float(w.y);
            }
        } else {
            L.st = p.n_src <= 32 ? make_float2(sx, sy) : *reinterpret_cast<const float2*>(src.stats + st_off);
            load_vec_any<E>(src.o + o_off + lane * E, L.ov);
        }
        if (src.keys) {
            const uint8_t* sc = scrambler_ptr(src.keys, p.keys_bstride, b, kh, D, 1);
            const float* ftab = reinterpret_cast<const float*>(sc);
            const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + 24 * D);
            load_vec_any<E>(ftab + kInvIn * D + lane * E, L.inv_in);
            load_vec_any<E>(ftab + kInvOut * D + lane * E, L.inv_out);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                L.p2[e] = utab[kP2 * D + lane * E + e];
                L.p1[e] = utab[kP1 * D + lane * E + e];
            }
        }
    };

    float out[E], acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] = acc[e] = 0.f;
    float denom = 0.f;
    const bool single = p.n_src == 1;
    bool pending = false;
    auto load_tables = [&](const uint8_t* keys, SrcLd<E>& L) {
        const uint8_t* sc = scrambler_ptr(keys, p.keys_bstride, b, kh, D, 1);
        const float* ftab = reinterpret_cast<const float*>(sc);
        const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + 24 * D);
        load_vec_any<E>(ftab + kInvIn * D + lane * E, L.inv_in);
        load_vec_any<E>(ftab + kInvOut * D + lane * E, L.inv_out);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            L.p2[e] = utab[kP2 * D + lane * E + e];
            L.p1[e] = utab[kP1 * D + lane * E + e];
        }
    };
    // quantised wire of O' (sda_unscramble_merge_quant): every key group's O' -- the domain's
    // normalised shard output, acc / its weight, still scrambled -- goes through
    // dequantize(quantize_affine(.)) before its unscramble (SCR_SHARD frames in quantN,
    // model.cpp:392, protocol.hpp:25-26). One tensor per (group, request, head): with one query row
    // the warp holds all of it; with more, a min / max pass (qpass 1) fills p.qscratch first.
    float gw = 0.f;   // the current group's weight
    int grp = 0;      // group index
    const int64_t n_bh = p.n_batch * p.q_heads;
    auto quant_group = [&](float* a) -> bool {   // false: min / max pass, nothing more to do
        if (p.quant_bits <= 0) return true;
        double lo = INFINITY, hi = -INFINITY;
        float y[E];
        const float iw = gw > 0.f ? 1.f / gw : 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            y[e] = a[e] * iw;
            lo = fmin(lo, (double)y[e]);
            hi = fmax(hi, (double)y[e]);
        }
        QParams q;
        if (p.q_rows == 1 || p.qpass == 1) {
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) {
                lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, m));
                hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, m));
            }
            if (p.qpass == 1) {
                if (lane == 0 && active && lo <= hi) {
                    atomicMin(p.qscratch + grp * n_bh + bh, dkey(lo));
                    atomicMax(p.qscratch + (p.n_groups + grp) * n_bh + bh, dkey(hi));
                }
                return false;
            }
            q = qparams_lohi(lo, hi, p.quant_bits);
        } else {
            q = qparams(p.qscratch + grp * n_bh, p.qscratch + (p.n_groups + grp) * n_bh, bh, p.quant_bits);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) a[e] = __double2float_rn(qround((double)y[e], q)) * gw;
        return true;
    };
    bool done_ll = false;
    if constexpr (E >= 2) {
    if (ll && p.n_src <= 32) {
        done_ll = true;
        // LL records: the words of up to 8 sources are requested at once and validated after,
        // instead of one blocking poll per word (the records are normally all there by now)
        constexpr int NB = 8, W = E / 2;   // 16-byte LL words per lane per source
        SrcLd<E> kt;
        for (int s0 = 0; s0 < p.n_src; s0 += NB) {
            uint4 raw[NB][W];
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                if (s0 + k < p.n_src) {
                    int64_t st_off, o_off;
                    offsets(p.src[s0 + k], st_off, o_off);
                    const uint8_t* rb = reinterpret_cast<const uint8_t*>(p.src[s0 + k].o) + 8 * (o_off + lane * E);
#pragma unroll
                    for (int m = 0; m < W; ++m)
                        asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(raw[k][m].x), "=r"(raw[k][m].y), "=r"(raw[k][m].z), "=r"(raw[k][m].w)
                                     : "l"(rb + 16 * m) : "memory");
                }
            }
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                const int s = s0 + k;
                if (s >= p.n_src) break;
                const K3Source& src = p.src[s];
                float ov[E];
#pragma unroll
                for (int m = 0; m < W; ++m) {
                    if (raw[k][m].y != ep || raw[k][m].w != ep) {   // not there yet: poll this word
                        int64_t st_off, o_off;
                        offsets(src, st_off, o_off);
                        const uint2 w2 = ll_load(reinterpret_cast<const uint8_t*>(src.o) + 8 * (o_off + lane * E) + 16 * m, ep);
                        raw[k][m].x = w2.x;
                        raw[k][m].z = w2.y;
                    }
                    ov[2 * m] = __uint_as_float(raw[k][m].x);
                    ov[2 * m + 1] = __uint_as_float(raw[k][m].z);
                }
                const float sx = __shfl_sync(0xffffffffu, st_lane.x, s & 31);
                const float sy = __shfl_sync(0xffffffffu, st_lane.y, s & 31);
                if (sy > 0.f) {
                    const float w = single ? 1.f : sy * expf(sx - mstar);
                    denom += single ? sy : w;
                    gw += w;
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[e] = fmaf(w, ov[e], acc[e]);
                    pending = true;
                }
                const bool group_end = (s + 1 == p.n_src) || (p.src[s + 1].keys != src.keys);
                if (group_end && pending && quant_group(acc)) {
                    if (src.keys) {
                        load_tables(src.keys, kt);
                        unscramble_acc<D>(kt, acc, out, sh, lane);
                    } else {
#pragma unroll
                        for (int e = 0; e < E; ++e) out[e] += acc[e];
                    }
                }
                if (group_end) {
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[e] = 0.f;
                    pending = false;
                    gw = 0.f;
                    ++grp;
                }
            }
        }
    }
    }
    if (!done_ll) {
        SrcLd<E> cur, nxt;
        load_src(0, cur);
        for (int s = 0; s < p.n_src; ++s) {
            if (s + 1 < p.n_src) load_src(s + 1, nxt);
            const K3Source& src = p.src[s];
            if (cur.st.y > 0.f) {
                const float w = single ? 1.f : cur.st.y * expf(cur.st.x - mstar);
                denom += single ? cur.st.y : w;
                gw += w;
    #pragma unroll
                for (int e = 0; e < E; ++e) acc[e] = fmaf(w, cur.ov[e], acc[e]);
                pending = true;
            }
            const bool group_end = (s + 1 == p.n_src) || (p.src[s + 1].keys != src.keys);
            if (group_end && pending && quant_group(acc)) {
                if (src.keys) {
                    unscramble_acc<D>(cur, acc, out, sh, lane);
                } else {
    #pragma unroll
                    for (int e = 0; e < E; ++e) out[e] += acc[e];
                }
            }
            if (group_end) {
    #pragma unroll
                for (int e = 0; e < E; ++e) acc[e] = 0.f;
                pending = false;
                gw = 0.f;
                ++grp;
            }
            cur = nxt;
        }
    }
    if (p.qpass == 1) return;   // the quantised wire's min / max pass stores nothing
    const bool masked = !(mstar > -INFINITY);
    if (masked && lane == 0 && p.err && active) atomicExch(p.err, (int32_t)SDA_ERR_MASKED_ROW);
    const float inv = masked ? __int_as_float(0x7fc00000) : (single ? 1.f : 1.f / denom);
#pragma unroll
    for (int e = 0; e < E; ++e) out[e] *= inv;
    const int64_t hr = (int64_t)h * p.q_rows + r;
    if (active)
        store_vec_any<E>(static_cast<TOut*>(p.out) + (p.out_bstride ? b * p.out_bstride + hr * D : row * D) + lane * E, out);
    if (p.out_stats && lane == 0 && active) {
        const int64_t so = p.out_bstride ? b * p.out_bstride + hr * 2 : row * 2;
        p.out_stats[so + 0] = single ? (masked ? -INFINITY : mstar) : mstar;
        p.out_stats[so + 1] = masked ? 0.f : denom;
    }
    if (ll && p.done_counter) {   // LL exchange: the last CTA opens the next step's epoch
        pdl_wait();   // ... once K2 (still serving other inquirers) has completed too
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(p.done_counter, 1u) == gridDim.x - 1) {
                *p.done_counter = 0;
                *p.epoch += 1;
            }
        }
    }
}

// Few sources (n_src <= kSmallSrc, plain memory): every source's stats and O' row are loaded up
// front, so a row costs ~2 dependent memory latencies (p_q^-1 index, then all data at once)
// instead of one per source -- the prefill merge (65K rows x 4 splits) is latency-bound on the
// per-row chain, not on bytes.
constexpr int kSmallSrc = 8;

template <int D, typename TOut, int NS, int RPW, bool EXACT>
__global__ void __launch_bounds__(128) k3_merge_small_kernel(const K3Params p) {
    constexpr int E = D / 32;
    __shared__ __align__(16) float sh_all[4][D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* sh = sh_all[warp];
    const int64_t total = p.n_batch * p.q_heads * p.q_rows;
    const int n = EXACT ? NS : p.n_src;   // !EXACT: n_src <= NS, guarded

    // RPW rows per warp, all of their sources' stats and O' rows in flight at once (NS = n_src
    // exactly; rows and their (b, h, r) decomposition fit 32 bits, checked by the launcher)
    int64_t rows[RPW], bs[RPW], rs[RPW];
    int hs[RPW];
    bool act[RPW];
    float2 st[RPW][NS];
    float ov[RPW][NS][E];
    const uint32_t qrows = (uint32_t)p.q_rows, qheads = (uint32_t)p.q_heads;
    SrcLd<E> kt0[RPW];   // the first key group's phi_V tables: inputs, read before the wait on K2
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const uint32_t row_raw = ((uint32_t)blockIdx.x * 4 + warp) * RPW + q;
        act[q] = row_raw < (uint32_t)total;
        const uint32_t row32 = act[q] ? row_raw : (uint32_t)total - 1;
        rows[q] = row32;
        const uint32_t bh = row32 / qrows;
        rs[q] = row32 - bh * qrows;
        const uint32_t b32 = bh / qheads;
        hs[q] = (int)(bh - b32 * qheads);
        bs[q] = b32;
        if (p.src[0].keys) {
            const uint8_t* sc = scrambler_ptr(p.src[0].keys, p.keys_bstride, bs[q], hs[q] / (p.q_heads / p.key_heads), D, 1);
            const float* ftab = reinterpret_cast<const float*>(sc);
            const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + kU16Off * D);
            load_vec_any<E>(ftab + kInvIn * D + lane * E, kt0[q].inv_in);
            load_vec_any<E>(ftab + kInvOut * D + lane * E, kt0[q].inv_out);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                kt0[q].p2[e] = utab[kP2 * D + lane * E + e];
                kt0[q].p1[e] = utab[kP1 * D + lane * E + e];
            }
        }
    }
    pdl_wait();   // launched early behind K2 (PDL): its partials must be complete
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int64_t bh = bs[q] * p.q_heads + hs[q];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (EXACT || s < n) {
                const K3Source& src = p.src[s];
                const int64_t ri = src.pq_inv ? (int64_t)src.pq_inv[bs[q] * p.pq_bstride + rs[q]] : rs[q];
                const int64_t hr = (int64_t)hs[q] * p.q_rows + ri;
                const int64_t st_off = src.bstride ? bs[q] * src.bstride + hr * 2 : (bh * p.q_rows + ri) * 2;
                const int64_t o_off = src.bstride ? bs[q] * src.bstride + hr * D : (bh * p.q_rows + ri) * D;
                st[q][s] = *reinterpret_cast<const float2*>(src.stats + st_off);
                load_vec_any<E>(src.o + o_off + lane * E, ov[q][s]);
            } else {
                st[q][s] = make_float2(-INFINITY, 0.f);
            }
        }
    }

#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int64_t b = bs[q], r = rs[q];
        const int h = hs[q];
        const int kh = h / (p.q_heads / p.key_heads);
        SrcLd<E> kt = kt0[q];
        auto load_tables = [&](const uint8_t* keys) {
            const uint8_t* sc = scrambler_ptr(keys, p.keys_bstride, b, kh, D, 1);
            const float* ftab = reinterpret_cast<const float*>(sc);
            const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + 24 * D);
            load_vec_any<E>(ftab + kInvIn * D + lane * E, kt.inv_in);
            load_vec_any<E>(ftab + kInvOut * D + lane * E, kt.inv_out);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                kt.p2[e] = utab[kP2 * D + lane * E + e];
                kt.p1[e] = utab[kP1 * D + lane * E + e];
            }
        };

        float mstar = -INFINITY;   // attention.cpp:103-105
#pragma unroll
        for (int s = 0; s < NS; ++s)
            if ((EXACT || s < n) && st[q][s].y > 0.f) mstar = fmaxf(mstar, st[q][s].x);

        float out[E], acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] = acc[e] = 0.f;
        float denom = 0.f;
        const bool single = n == 1;
        bool pending = false;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (EXACT || s < n) {
                const K3Source& src = p.src[s];
                if (s > 0 && src.keys && src.keys != p.src[s - 1].keys) load_tables(src.keys);   // new group
                if (st[q][s].y > 0.f) {
                    const float w = single ? 1.f : st[q][s].y * expf(st[q][s].x - mstar);
                    denom += single ? st[q][s].y : w;
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[e] = fmaf(w, ov[q][s][e], acc[e]);
                    pending = true;
                }
                const bool group_end = (s + 1 == n) || (p.src[s + 1].keys != src.keys);
                if (group_end && pending) {
                    if (src.keys) {
                        unscramble_acc<D>(kt, acc, out, sh, lane);
                    } else {
#pragma unroll
                        for (int e = 0; e < E; ++e) out[e] += acc[e];
                    }
#pragma unroll
                    for (int e = 0; e < E; ++e) acc[e] = 0.f;
                    pending = false;
                }
            }
        }
        const bool masked = !(mstar > -INFINITY);
        if (masked && lane == 0 && p.err && act[q]) atomicExch(p.err, (int32_t)SDA_ERR_MASKED_ROW);
        const float inv = masked ? __int_as_float(0x7fc00000) : (single ? 1.f : 1.f / denom);
#pragma unroll
        for (int e = 0; e < E; ++e) out[e] *= inv;
        const int64_t hr = (int64_t)h * p.q_rows + r;
        if (act[q])
            store_vec_any<E>(static_cast<TOut*>(p.out) + (p.out_bstride ? b * p.out_bstride + hr * D : rows[q] * D) +
                                 lane * E, out);
        if (p.out_stats && lane == 0 && act[q]) {
            const int64_t so = p.out_bstride ? b * p.out_bstride + hr * 2 : rows[q] * 2;
            p.out_stats[so + 0] = single ? (masked ? -INFINITY : mstar) : mstar;
            p.out_stats[so + 1] = masked ? 0.f : denom;
        }
    }
}

// fwht_group over U independent rows at once (lane owns elements [lane*E, lane*E+E) of each):
// every stage runs across all rows before the next, so the shuffle latencies overlap
// (E = 4: the butterflies as packed f32x2 adds / FMAs -- the kernel is issue-bound)
__device__ __forceinline__ uint64_t k3_f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void k3_split(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t k3_add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t k3_sub2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t k3_fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
template <int U, int E>
__device__ __forceinline__ void fwht_rows(float (&v)[U][E], int lane) {
    if constexpr (E == 4) {
#pragma unroll
        for (int u = 0; u < U; ++u) {   // (0,1) (2,3), then (0,2) (1,3): the same sums in the same order
            const uint64_t a = k3_f2(v[u][0], v[u][2]), b = k3_f2(v[u][1], v[u][3]);
            float s0, s1, d0, d1;
            k3_split(k3_add2(a, b), s0, s1);   // v0 + v1, v2 + v3
            k3_split(k3_sub2(a, b), d0, d1);   // v0 - v1, v2 - v3
            const uint64_t a2 = k3_f2(s0, d0), b2 = k3_f2(s1, d1);
            k3_split(k3_add2(a2, b2), v[u][0], v[u][1]);
            k3_split(k3_sub2(a2, b2), v[u][2], v[u][3]);
        }
    } else {
#pragma unroll
        for (int h = 1; h < E; h <<= 1)
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < E; ++i)
                    if ((i & h) == 0) {
                        const float a = v[u][i], b = v[u][i + h];
                        v[u][i] = a + b;
                        v[u][i + h] = a - b;
                    }
    }
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
        const float sgn = (lane & m) ? -1.f : 1.f;
        float o[U][E];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < E; ++i) o[u][i] = __shfl_xor_sync(0xffffffffu, v[u][i], m);
        if constexpr (E % 2 == 0) {
            const uint64_t sg2 = k3_f2(sgn, sgn);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < E; i += 2)
                    k3_split(k3_fma2(k3_f2(v[u][i], v[u][i + 1]), sg2, k3_f2(o[u][i], o[u][i + 1])), v[u][i], v[u][i + 1]);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < E; ++i) v[u][i] = fmaf(sgn, v[u][i], o[u][i]);
        }
    }
}

// x[k & (E-1)] for a run-time k as a tree of E-1 selects on k's bits (keeps x in registers)
template <int E>
__device__ __forceinline__ float pick(const float* x, uint32_t k) {
    if constexpr (E == 1) {
        return x[0];
    } else {
        const float lo = pick<E / 2>(x, k), hi = pick<E / 2>(x + E / 2, k);
        return (k & (E / 2)) ? hi : lo;
    }
}

// Prefill-shaped merge (q_rows >= 64, plain memory, <= 8 sources): a CTA owns 64 consecutive
// rows of one (request, head), so the phi_V^-1 tables of its sources are staged in shared memory
// once per CTA (k3_merge_small_kernel re-reads them from L1 for every row: the u16 permutation
// loads alone were most of its L1 traffic). Per row: coalesced 16-byte loads of every source's O'
// row, the weighted sum in scrambled space per key group, and one unscramble per group through the
// warp's shared-memory row (P2 gather -> 2 register + 5 shuffle butterfly stages -> P1 gather),
// then coalesced stores. Both gathers follow the key image's schedules (kSchedOff): every load
// instruction's 32 addresses fall in 32 distinct banks, so a gather costs E wavefronts, not the
// ~2E a random permutation's collisions cost. The p_q^-1 row indices of a warp's 16 rows are fetched in one load per
// source up front, and U rows' stats and O' of every source are requested before any is used.
template <int D, typename TOut, int NS, bool EXACT>
__global__ void __launch_bounds__(128) k3_rows_kernel(const K3Params p) {
    constexpr int E = D / 32;
    constexpr int U = NS >= 4 ? 1 : 4 / NS;   // rows in flight per warp
    constexpr int RPW = 16;                    // rows per warp; 64 per CTA
    __shared__ __align__(16) float s_in[NS][D];    // InvIn (1 / s2)
    __shared__ __align__(16) float s_out[NS][D];   // InvOut (1 / (s1 sqrt(d)))
    // the two gathers of the unscramble in the key set's bank-conflict-free order (keys.cpp
    // gather_schedule): load k of lane l reads address s_g2[s][k*32+l] (the 32 addresses of a load
    // hit 32 different banks); element e of the lane's E is the value of load (s_k2[s][l] >> 4e) & 15
    __shared__ __align__(16) uint16_t s_g2[NS][D], s_g1[NS][D];
    __shared__ uint32_t s_k2[NS][32], s_k1[NS][32];
    __shared__ __align__(16) float s_row[4][U][D];
    const int n = EXACT ? NS : p.n_src;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bh = blockIdx.y;
    const int h = (int)(bh % p.q_heads);
    const int64_t b = bh / p.q_heads;
    const int kh = h / (p.q_heads / p.key_heads);
    for (int s = 0; s < n; ++s) {
        if (!p.src[s].keys) continue;
        const uint8_t* sc = scrambler_ptr(p.src[s].keys, p.keys_bstride, b, kh, D, 1);
        const float* ftab = reinterpret_cast<const float*>(sc);
        const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + 24 * D);
        const uint8_t* sch = sc + kSchedOff * D;
        for (int j = threadIdx.x; j < D; j += blockDim.x) {
            s_in[s][j] = ftab[kInvIn * D + j];
            s_out[s][j] = ftab[kInvOut * D + j];
            const int l = j / E, k = j % E;   // schedule entry (lane l, load k) -> slot k*32 + l
            s_g2[s][k * 32 + l] = utab[kP2 * D + l * E + sch[kSchedP2 * D + j]];
            s_g1[s][k * 32 + l] = utab[kP1 * D + l * E + sch[kSchedP1 * D + j]];
        }
        for (int l = threadIdx.x; l < 32; l += blockDim.x) {
            uint32_t k2 = 0, k1 = 0;
            for (int k = 0; k < E; ++k) {
                k2 |= (uint32_t)k << (4 * sch[kSchedP2 * D + l * E + k]);
                k1 |= (uint32_t)k << (4 * sch[kSchedP1 * D + l * E + k]);
            }
            s_k2[s][l] = k2;
            s_k1[s][l] = k1;
        }
    }
    pdl_wait();   // launched early behind K2 (PDL): its partials must be complete
    __syncthreads();

    const int64_t r_base = (int64_t)blockIdx.x * (4 * RPW) + warp * RPW;
    uint32_t ridx[NS];   // lane t < RPW: source s's O' row for output row r_base + t
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        ridx[s] = 0;
        if ((EXACT || s < n) && lane < RPW && r_base + lane < p.q_rows)
            ridx[s] = p.src[s].pq_inv ? p.src[s].pq_inv[b * p.pq_bstride + r_base + lane] : (uint32_t)(r_base + lane);
    }
    // per-source bases of this (request, head): a row is then one 32-bit multiply-add away
    const float* obase[NS];
    const float* sbase[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const K3Source& src = p.src[s];
        const int64_t off = src.bstride ? b * src.bstride + (int64_t)h * p.q_rows * D : bh * p.q_rows * D;
        const int64_t soff = src.bstride ? b * src.bstride + (int64_t)h * p.q_rows * 2 : bh * p.q_rows * 2;
        obase[s] = (EXACT || s < n) ? src.o + off : nullptr;
        sbase[s] = (EXACT || s < n) ? src.stats + soff : nullptr;
    }
    TOut* const obh = static_cast<TOut*>(p.out) + (p.out_bstride ? b * p.out_bstride + (int64_t)h * p.q_rows * D : bh * p.q_rows * D);
    float* const sbh = p.out_stats ? p.out_stats + (p.out_bstride ? b * p.out_bstride + (int64_t)h * p.q_rows * 2 : bh * p.q_rows * 2)
                                   : nullptr;
    float* rows[U];
#pragma unroll
    for (int u = 0; u < U; ++u) rows[u] = s_row[warp][u];
    const bool single = n == 1;
    for (int t0 = 0; t0 < RPW; t0 += U) {
        float2 st[U][NS];
        float xv[U][NS][E];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool valid = r_base + t0 + u < p.q_rows;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const uint32_t ri = __shfl_sync(0xffffffffu, ridx[s], t0 + u);
                if ((EXACT || s < n) && valid) {
                    st[u][s] = *reinterpret_cast<const float2*>(sbase[s] + (size_t)ri * 2);
                    load_vec_any<E>(obase[s] + (size_t)ri * D + lane * E, xv[u][s]);
                } else {
                    st[u][s] = make_float2(-INFINITY, 0.f);
#pragma unroll
                    for (int e = 0; e < E; ++e) xv[u][s][e] = 0.f;
                }
            }
        }
        // the U rows go through every step together (one loop nest per step), so their shared-memory
        // round trips and shuffle stages overlap instead of forming U dependent chains
        float mstar[U], denom[U], acc[U][E], out[U][E];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            mstar[u] = -INFINITY;   // attention.cpp:103-105
#pragma unroll
            for (int s = 0; s < NS; ++s)
                if ((EXACT || s < n) && st[u][s].y > 0.f) mstar[u] = fmaxf(mstar[u], st[u][s].x);
            denom[u] = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[u][e] = out[u][e] = 0.f;
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (!(EXACT || s < n)) continue;
            const K3Source& src = p.src[s];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                // a source with no visible key (exp_sum 0) adds nothing: a zero weight rather than a
                // branch, so the unscramble below stays warp-uniform code
                const bool live = st[u][s].y > 0.f;
                const float w = live ? (single ? 1.f : st[u][s].y * expf(st[u][s].x - mstar[u])) : 0.f;
                denom[u] += single ? st[u][s].y : w;
#pragma unroll
                for (int e = 0; e < E; ++e) acc[u][e] = live ? fmaf(w, xv[u][s][e], acc[u][e]) : acc[u][e];   // never 0 * NaN
            }
            const bool group_end = (s + 1 == n) || (p.src[s + 1].keys != src.keys);
            if (!group_end) continue;
            if (src.keys) {   // one unscramble per key group (linearity)
                // t = acc / s2 ; u[j] = t[P2[j]] ; w = H u ; y[i] = w[P1[i]] / (s1[i] sqrt(d))
                float tin[E], tout[E], v[U][E], x[E];
                int g2[E], g1[E];
                load_vec_any<E>(&s_in[s][lane * E], tin);
                load_vec_any<E>(&s_out[s][lane * E], tout);
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    g2[k] = s_g2[s][k * 32 + lane];
                    g1[k] = s_g1[s][k * 32 + lane];
                }
                const uint32_t k2 = s_k2[s][lane], k1 = s_k1[s][lane];
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int e = 0; e < E; ++e) v[u][e] = acc[u][e] * tin[e];
                    store_vec_any<E>(rows[u] + lane * E, v[u]);
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < U; ++u) {   // u[j] = t[P2[j]] over conflict-free loads
#pragma unroll
                    for (int k = 0; k < E; ++k) x[k] = rows[u][g2[k]];
#pragma unroll
                    for (int e = 0; e < E; ++e) v[u][e] = pick<E>(x, k2 >> (4 * e));
                }
                fwht_rows<U, E>(v, lane);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < U; ++u) store_vec_any<E>(rows[u] + lane * E, v[u]);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < U; ++u) {   // y[i] = w[P1[i]] InvOut[i]
#pragma unroll
                    for (int k = 0; k < E; ++k) x[k] = rows[u][g1[k]];
#pragma unroll
                    for (int e = 0; e < E; ++e) out[u][e] = fmaf(pick<E>(x, k1 >> (4 * e)), tout[e], out[u][e]);
                }
                __syncwarp();
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int e = 0; e < E; ++e) out[u][e] += acc[u][e];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < E; ++e) acc[u][e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = r_base + t0 + u;
            const bool valid = r < p.q_rows;
            const bool masked = !(mstar[u] > -INFINITY);
            if (masked && lane == 0 && p.err && valid) atomicExch(p.err, (int32_t)SDA_ERR_MASKED_ROW);
            const float inv = masked ? __int_as_float(0x7fc00000) : (single ? 1.f : 1.f / denom[u]);
#pragma unroll
            for (int e = 0; e < E; ++e) out[u][e] *= inv;
            if (valid) {
                store_vec_any<E>(obh + (size_t)r * D + lane * E, out[u]);
                if (sbh && lane == 0)
                    *reinterpret_cast<float2*>(sbh + (size_t)r * 2) =
                        make_float2(single ? (masked ? -INFINITY : mstar[u]) : mstar[u], masked ? 0.f : denom[u]);
            }
        }
    }
}

template <int D, typename TOut, int NS, bool EXACT = true>
static cudaError_t launch_k3_rows(const K3Params& p, cudaStream_t st) {
    const dim3 grid((unsigned)((p.q_rows + 63) / 64), (unsigned)(p.n_batch * p.q_heads));
    return pdl_launch(k3_rows_kernel<D, TOut, NS, EXACT>, grid, dim3(128), st, p);
}

template <int D, typename TOut, int NS, bool EXACT = true>
static void launch_k3_small(const K3Params& p, int64_t total, cudaStream_t st) {
    constexpr int RPW = NS * (D / 32) <= 16 ? 2 : 1;   // in-flight rows per warp (4 measured slower)
    const int64_t per_cta = 4 * RPW;
    pdl_launch(k3_merge_small_kernel<D, TOut, NS, RPW, EXACT>, dim3((unsigned)((total + per_cta - 1) / per_cta)), dim3(128),
               st, p);
}

template <int D, typename TOut>
static cudaError_t launch_k3_t(const K3Params& p, cudaStream_t st) {
    const int64_t total = p.n_batch * p.q_heads * p.q_rows;
    if (p.quant_bits > 0) {   // quantised O' wire: the general form (min / max pass first for > 1 row)
        const dim3 grid((unsigned)((total + 3) / 4));
        if (p.q_rows > 1) {
            const int64_t n = (int64_t)p.n_groups * p.n_batch * p.q_heads;
            cudaError_t e = cudaMemsetAsync(p.qscratch, 0xFF, n * 8, st);
            if (e == cudaSuccess) e = cudaMemsetAsync(p.qscratch + n, 0x00, n * 8, st);
            if (e != cudaSuccess) return e;
            K3Params p1 = p;
            p1.qpass = 1;
            if ((e = pdl_launch(k3_merge_kernel<D, TOut>, grid, dim3(128), st, p1)) != cudaSuccess) return e;
        }
        K3Params p2 = p;
        p2.qpass = 2;
        return pdl_launch(k3_merge_kernel<D, TOut>, grid, dim3(128), st, p2);
    }
    if (p.ll) return pdl_launch(k3_merge_kernel<D, TOut>, dim3((unsigned)((total + 3) / 4)), dim3(128), st, p);
    const bool small_ok = total < (int64_t(1) << 30) && !getenv("SDA_K3_PIPELINED");
    // prefill-shaped merges of one key group (+ plaintext): the tensor-core form (k3_tc.cu) where
    // it measured faster than the rows kernel -- three or more sources (tools/k3_bench.py: the C5
    // chunk's 2 splits + own span 82 vs 104 us; with 1-2 sources the rows kernel's 7 CTAs per SM
    // hide the gathers' latency better than the TC form's single CTA). SDA_K3_TC=1 forces it.
    if (!getenv("SDA_K3_NO_TC") && (p.n_src >= 3 || getenv("SDA_K3_TC"))) {
        const cudaError_t e = launch_k3_tc(p, D, std::is_same<TOut, float>::value ? SDA_F32 : SDA_BF16, st);
        if (e != cudaErrorNotSupported) return e;
    }
    // prefill-shaped rows (many per (request, head)): the table-staging row kernel
    // (1-2 sources; with more, a warp's U = 1 row in flight loses to the preload kernel's 2 rows
    // x all sources in flight: 4 splits 82 vs 55 us, tools/k3_bench.py; SDA_K3_ROWS=1 forces it)
    if (p.q_rows >= 64 && p.n_batch * p.q_heads < 65536 && !getenv("SDA_K3_NO_ROWS") &&
        (p.n_src <= 2 || (getenv("SDA_K3_ROWS") && p.n_src <= kSmallSrc))) {
        switch (p.n_src) {
            case 1: return launch_k3_rows<D, TOut, 1>(p, st);
            case 2: return launch_k3_rows<D, TOut, 2>(p, st);
            case 3: case 4: return launch_k3_rows<D, TOut, 4, false>(p, st);
            default: return launch_k3_rows<D, TOut, 8, false>(p, st);
        }
    }
    if constexpr (D <= 128) {   // 9..16 sources (the decode split fold): all in flight, one row per warp
        if (small_ok && p.n_src > kSmallSrc && p.n_src <= 16) {
            launch_k3_small<D, TOut, 16, false>(p, total, st);
            return cudaGetLastError();
        }
    }
    if (p.n_src <= kSmallSrc && small_ok) {
        switch (p.n_src) {
            case 1: launch_k3_small<D, TOut, 1>(p, total, st); break;
            case 2: launch_k3_small<D, TOut, 2>(p, total, st); break;
            case 3: launch_k3_small<D, TOut, 3>(p, total, st); break;
            case 4: launch_k3_small<D, TOut, 4>(p, total, st); break;
            case 5: launch_k3_small<D, TOut, 5>(p, total, st); break;
            case 6: launch_k3_small<D, TOut, 6>(p, total, st); break;
            case 7: launch_k3_small<D, TOut, 7>(p, total, st); break;
            default: launch_k3_small<D, TOut, 8>(p, total, st); break;
        }
    } else {
        return pdl_launch(k3_merge_kernel<D, TOut>, dim3((unsigned)((total + 3) / 4)), dim3(128), st, p);
    }
    return cudaGetLastError();
}

SDA_SPIN_ACCESSOR(spin_access_k3_merge)

// Small head dims (d in {4, 8, 16}: the reference's own model / protocol tests, test_model.cpp:17-19,
// helpers.hpp:19): one thread per output row, the whole row and the phi_V^-1 of its group in the
// thread's registers / local memory. Same two passes and the same per-group unscramble as
// k3_merge_kernel (no LL records: the LL exchange is a d >= 64 decode form).
template <int D, typename TOut>
__global__ void __launch_bounds__(128) k3_merge_tiny_kernel(const K3Params p) {
    pdl_wait();
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
    float mstar = -INFINITY;   // attention.cpp:103-105
    for (int s = 0; s < p.n_src; ++s) {
        int64_t so, oo;
        offs(p.src[s], so, oo);
        const float2 st = *reinterpret_cast<const float2*>(p.src[s].stats + so);
        if (st.y > 0.f) mstar = fmaxf(mstar, st.x);
    }
    const bool single = p.n_src == 1;
    float out[D], acc[D];
#pragma unroll
    for (int e = 0; e < D; ++e) out[e] = acc[e] = 0.f;
    float denom = 0.f;
    bool pending = false;
    for (int s = 0; s < p.n_src; ++s) {
        const K3Source& src = p.src[s];
        int64_t so, oo;
        offs(src, so, oo);
        const float2 st = *reinterpret_cast<const float2*>(src.stats + so);
        if (st.y > 0.f) {
            const float w = single ? 1.f : st.y * expf(st.x - mstar);
            denom += single ? st.y : w;
#pragma unroll
            for (int e = 0; e < D; ++e) acc[e] = fmaf(w, src.o[oo + e], acc[e]);
            pending = true;
        }
        const bool group_end = (s + 1 == p.n_src) || (p.src[s + 1].keys != src.keys);
        if (group_end && pending) {
            if (src.keys) {
                // u[j] = acc[P2[j]] / s2[P2[j]] ; w = H u ; y[i] = w[P1[i]] / (s1[i] sqrt(d))
                const uint8_t* sc = scrambler_ptr(src.keys, p.keys_bstride, b, kh, D, 1);
                const float* ftab = reinterpret_cast<const float*>(sc);
                const uint16_t* utab = reinterpret_cast<const uint16_t*>(sc + 24 * D);
                float t[D], u[D];
#pragma unroll
                for (int e = 0; e < D; ++e) t[e] = acc[e] * ftab[kInvIn * D + e];
                for (int j = 0; j < D; ++j) u[j] = t[utab[kP2 * D + j]];
#pragma unroll
                for (int hh = 1; hh < D; hh <<= 1)
#pragma unroll
                    for (int i = 0; i < D; ++i)
                        if ((i & hh) == 0) {
                            const float a = u[i], c = u[i + hh];
                            u[i] = a + c;
                            u[i + hh] = a - c;
                        }
                for (int i = 0; i < D; ++i) out[i] += u[utab[kP1 * D + i]] * ftab[kInvOut * D + i];
            } else {
#pragma unroll
                for (int e = 0; e < D; ++e) out[e] += acc[e];
            }
#pragma unroll
            for (int e = 0; e < D; ++e) acc[e] = 0.f;
            pending = false;
        }
    }
    const bool masked = !(mstar > -INFINITY);
    if (masked && p.err) atomicExch(p.err, (int32_t)SDA_ERR_MASKED_ROW);
    const float inv = masked ? __int_as_float(0x7fc00000) : (single ? 1.f : 1.f / denom);
#pragma unroll
    for (int e = 0; e < D; ++e) out[e] *= inv;
    const int64_t hr = (int64_t)h * p.q_rows + r;
    TOut* o = static_cast<TOut*>(p.out) + (p.out_bstride ? b * p.out_bstride + hr * D : row * D);
#pragma unroll
    for (int e = 0; e < D; ++e) o[e] = (TOut)out[e];
    if (p.out_stats) {
        const int64_t so = p.out_bstride ? b * p.out_bstride + hr * 2 : row * 2;
        p.out_stats[so + 0] = single ? (masked ? -INFINITY : mstar) : mstar;
        p.out_stats[so + 1] = masked ? 0.f : denom;
    }
}

template <int D, typename TOut>
static cudaError_t launch_k3_tiny(const K3Params& p, cudaStream_t st) {
    if (p.ll) return cudaErrorInvalidValue;
    const int64_t total = p.n_batch * p.q_heads * p.q_rows;
    return pdl_launch(k3_merge_tiny_kernel<D, TOut>, dim3((unsigned)((total + 127) / 128)), dim3(128), st, p);
}

cudaError_t launch_k3(const K3Params& p, int d, int odt, cudaStream_t st) {
    const bool bf = odt == SDA_BF16;
    switch (d) {
        case 4: return bf ? launch_k3_tiny<4, __nv_bfloat16>(p, st) : launch_k3_tiny<4, float>(p, st);
        case 8: return bf ? launch_k3_tiny<8, __nv_bfloat16>(p, st) : launch_k3_tiny<8, float>(p, st);
        case 16: return bf ? launch_k3_tiny<16, __nv_bfloat16>(p, st) : launch_k3_tiny<16, float>(p, st);
        case 32: return bf ? launch_k3_t<32, __nv_bfloat16>(p, st) : launch_k3_t<32, float>(p, st);
        case 64: return bf ? launch_k3_t<64, __nv_bfloat16>(p, st) : launch_k3_t<64, float>(p, st);
        case 128: return bf ? launch_k3_t<128, __nv_bfloat16>(p, st) : launch_k3_t<128, float>(p, st);
        case 256: return bf ? launch_k3_t<256, __nv_bfloat16>(p, st) : launch_k3_t<256, float>(p, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sda
