// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat extern "C" surface over the reference's own hot-path functions so
// that Python tests (ctypes) and bench.py's reference arm can call the
// UNMODIFIED reference implementation. It is compiled by oracle/Makefile
// together with the reference sources straight from /root/reference (no
// source is copied into this repo) into oracle/_ref/libsdattn_ref.so.
//
// Nothing here is shipped: the product library never links this file.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "sdattn/attention.hpp"
#include "sdattn/quant.hpp"
#include "sdattn/frame.hpp"
#include "sdattn/float_format.hpp"
#include "sdattn/fwht.hpp"
#include "sdattn/model.hpp"
#include "sdattn/permutation.hpp"
#include "sdattn/rng.hpp"
#include "sdattn/scrambler.hpp"

using namespace sdattn;

namespace {

Matrix to_matrix(const double* p, std::size_t r, std::size_t c) {
    return Matrix(r, c, std::vector<double>(p, p + r * c));
}

void from_matrix(const Matrix& m, double* out) { std::memcpy(out, m.data.data(), sizeof(double) * m.data.size()); }

Scrambler make_scrambler(std::size_t d, const double* s1, const std::uint32_t* p1,
                         const std::uint32_t* p2, const double* s2) {
    Scrambler s;
    s.dim = d;
    s.s1.factors.assign(s1, s1 + d);
    s.s2.factors.assign(s2, s2 + d);
    s.p1.forward.assign(p1, p1 + d);
    s.p2.forward.assign(p2, p2 + d);
    return s;
}

void put_scrambler(const Scrambler& s, double* s1, std::uint32_t* p1, std::uint32_t* p2, double* s2) {
    std::memcpy(s1, s.s1.factors.data(), sizeof(double) * s.dim);
    std::memcpy(s2, s.s2.factors.data(), sizeof(double) * s.dim);
    std::memcpy(p1, s.p1.forward.data(), sizeof(std::uint32_t) * s.dim);
    std::memcpy(p2, s.p2.forward.data(), sizeof(std::uint32_t) * s.dim);
}

KeySetSpec make_spec(std::uint64_t request_id, std::uint32_t layer, std::uint32_t domain,
                     std::size_t n_heads, std::size_t d, double lo, double hi, int mode,
                     std::size_t l_q, std::size_t l_k) {
    KeySetSpec spec;
    spec.request_id = request_id;
    spec.layer = layer;
    spec.domain = domain;
    spec.n_heads = n_heads;
    spec.head_dim = d;
    spec.mag_lo = lo;
    spec.mag_hi = hi;
    spec.mode = mode == 1 ? ScramblerMode::s1_only : ScramblerMode::s1_and_s2;
    spec.l_q = l_q;
    spec.l_k = l_k;
    return spec;
}

}  // namespace

extern "C" {

void ref_rng_u64(std::uint64_t seed, std::size_t n, std::uint64_t* out) {
    RngStream r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void ref_rng_gaussian(std::uint64_t seed, std::size_t n, double* out) {
    RngStream r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.next_gaussian();
}

std::uint64_t ref_derive_seed(std::uint64_t base, const std::uint64_t* tags, std::size_t n) {
    // derive_seed takes an initializer_list; fold one tag at a time, which the
    // reference defines as the same chain (rng.cpp:35-39).
    std::uint64_t s = base;
    for (std::size_t i = 0; i < n; ++i) s = derive_seed(s, {tags[i]});
    return s;
}

int ref_random_permutation(std::size_t n, std::uint64_t seed, std::uint32_t* out) {
    try {
        RngStream r(seed);
        Permutation p = random_permutation(n, r);
        std::memcpy(out, p.forward.data(), sizeof(std::uint32_t) * n);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

double ref_round_to_format(double x, int fmt) { return round_to_format(x, static_cast<FloatFormat>(fmt)); }

int ref_fwht(double* x, std::size_t n) {
    try {
        fwht_normalized_inplace(std::span<double>(x, n));
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_build_scrambler(std::size_t d, double lo, double hi, std::uint64_t seed, int mode, double* s1,
                        std::uint32_t* p1, std::uint32_t* p2, double* s2) {
    try {
        RngStream r(seed);
        Scrambler s = build_scrambler(d, lo, hi, r, mode == 1 ? ScramblerMode::s1_only : ScramblerMode::s1_and_s2);
        put_scrambler(s, s1, p1, p2, s2);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Keyset: kq_* / v_* are [n_heads][d]; p_q [l_q], p_kv [l_k].
int ref_negotiate_keyset(std::uint64_t shared_seed, std::uint64_t request_id, std::uint32_t layer,
                         std::uint32_t domain, std::size_t n_heads, std::size_t d, double lo, double hi,
                         int mode, std::size_t l_q, std::size_t l_k, double* kq_s1, std::uint32_t* kq_p1,
                         std::uint32_t* kq_p2, double* kq_s2, double* v_s1, std::uint32_t* v_p1,
                         std::uint32_t* v_p2, double* v_s2, std::uint32_t* p_q, std::uint32_t* p_kv,
                         std::uint64_t* token_perm_seed) {
    try {
        ScramblerKeySet ks = negotiate_keyset(shared_seed, make_spec(request_id, layer, domain, n_heads, d, lo,
                                                                     hi, mode, l_q, l_k));
        for (std::size_t h = 0; h < n_heads; ++h) {
            put_scrambler(ks.phi_kq[h], kq_s1 + h * d, kq_p1 + h * d, kq_p2 + h * d, kq_s2 + h * d);
            put_scrambler(ks.phi_v[h], v_s1 + h * d, v_p1 + h * d, v_p2 + h * d, v_s2 + h * d);
        }
        if (p_q) std::memcpy(p_q, ks.p_q.forward.data(), sizeof(std::uint32_t) * l_q);
        if (p_kv) std::memcpy(p_kv, ks.p_kv.forward.data(), sizeof(std::uint32_t) * l_k);
        *token_perm_seed = ks.token_perm_seed;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_span_perm(std::uint64_t token_perm_seed, std::uint64_t tag, std::uint64_t first_pos, std::size_t len,
                  std::uint32_t* out) {
    try {
        ScramblerKeySet ks;
        ks.token_perm_seed = token_perm_seed;
        Permutation p = ks.span_perm(tag, first_pos, len);
        std::memcpy(out, p.forward.data(), sizeof(std::uint32_t) * len);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// variant: 0 apply_phi, 1 apply_phi_inv_t, 2 apply_phi_inv
int ref_apply_phi(const double* x, std::size_t rows, std::size_t d, const double* s1, const std::uint32_t* p1,
                  const std::uint32_t* p2, const double* s2, int variant, double* out) {
    try {
        const Scrambler s = make_scrambler(d, s1, p1, p2, s2);
        const Matrix m = to_matrix(x, rows, d);
        Matrix y = variant == 0 ? apply_phi(m, s) : variant == 1 ? apply_phi_inv_t(m, s) : apply_phi_inv(m, s);
        from_matrix(y, out);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_shard_attention(const double* q, std::size_t lq, const double* k, const double* v, std::size_t lk,
                        std::size_t d, int mask_kind, std::int64_t offset, double* out, double* row_max,
                        double* exp_sum) {
    try {
        AttentionMask mask = mask_kind == 1 ? AttentionMask::causal(offset) : AttentionMask::none();
        AttentionShard s = shard_attention(to_matrix(q, lq, d), to_matrix(k, lk, d), to_matrix(v, lk, d), mask, d);
        from_matrix(s.output, out);
        std::memcpy(row_max, s.stats.row_max.data(), sizeof(double) * lq);
        std::memcpy(exp_sum, s.stats.exp_sum.data(), sizeof(double) * lq);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

int ref_merge_shards(std::size_t n, const double* const* outs, const double* const* rmax,
                     const double* const* esum, std::size_t rows, std::size_t cols, double* merged) {
    try {
        std::vector<AttentionShard> shards(n);
        for (std::size_t i = 0; i < n; ++i) {
            shards[i].output = to_matrix(outs[i], rows, cols);
            shards[i].stats.row_max.assign(rmax[i], rmax[i] + rows);
            shards[i].stats.exp_sum.assign(esum[i], esum[i] + rows);
        }
        from_matrix(merge_shards(shards), merged);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// dec_output with the phi_v of `head` from a keyset (shared_seed + spec) and
// p_q = span_perm(0, q_first_pos, lq).
int ref_dec_output(std::uint64_t shared_seed, std::uint64_t request_id, std::uint32_t layer, std::uint32_t domain,
                   std::size_t n_heads, std::size_t d, double lo, double hi, int mode, std::size_t head,
                   std::uint64_t q_first_pos, const double* o_s, const double* rmax_s, const double* esum_s,
                   std::size_t lq, double* out, double* rmax, double* esum) {
    try {
        ScramblerKeySet ks =
            negotiate_keyset(shared_seed, make_spec(request_id, layer, domain, n_heads, d, lo, hi, mode, 1, 1));
        ks.p_q = ks.span_perm(0, q_first_pos, lq);
        ShardStats st;
        st.row_max.assign(rmax_s, rmax_s + lq);
        st.exp_sum.assign(esum_s, esum_s + lq);
        AttentionShard r = dec_output(to_matrix(o_s, lq, d), st, ks, head);
        from_matrix(r.output, out);
        std::memcpy(rmax, r.stats.row_max.data(), sizeof(double) * lq);
        std::memcpy(esum, r.stats.exp_sum.data(), sizeof(double) * lq);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// One (request, head) of the scrambled decode/prefill step composed exactly
// as the reference's protocol does it (protocol.cpp:876-899 Q scramble,
// :987-1016 K/V scramble, :1053-1104 keyless partial attention,
// :921-949 dec + merge), with wire rounding `wire_fmt` applied to Q', K', V'
// (model.cpp:387-389). O' and the stats are kept in f64 ("rounding-matched
// oracle": the device keeps them in f32).
//   q: [lq x d]; k, v: [n_nodes][lk x d] (plaintext shards); node n is domain
//   n+1 with shard first_pos = n*lk.  out: [lq x d].
int ref_scrambled_step(std::uint64_t shared_seed, std::uint64_t request_id, std::uint32_t layer,
                       std::size_t n_heads, std::size_t head, std::size_t d, double lo, double hi, int mode,
                       int wire_fmt, std::size_t n_nodes, const double* q, std::size_t lq,
                       std::uint64_t q_first_pos, const double* k, const double* v, std::size_t lk, double* out) {
    try {
        const FloatFormat wf = static_cast<FloatFormat>(wire_fmt);
        const Matrix qm = to_matrix(q, lq, d);
        std::vector<AttentionShard> shards;
        for (std::size_t n = 0; n < n_nodes; ++n) {
            ScramblerKeySet ks = negotiate_keyset(
                shared_seed, make_spec(request_id, layer, static_cast<std::uint32_t>(n + 1), n_heads, d, lo, hi, mode, 1, 1));
            ks.p_q = ks.span_perm(0, q_first_pos, lq);
            ks.p_kv = ks.span_perm(1, n * lk, lk);
            ScrambledTriple t = enc_qkv(qm, to_matrix(k + n * lk * d, lk, d), to_matrix(v + n * lk * d, lk, d), ks, head);
            t.q_s = round_to_format(t.q_s, wf);
            t.k_s = round_to_format(t.k_s, wf);
            t.v_s = round_to_format(t.v_s, wf);
            AttentionShard scr = scrambled_shard_attention(t, AttentionMask::none(), d);
            shards.push_back(dec_output(scr.output, scr.stats, ks, head));
        }
        from_matrix(merge_shards(shards), out);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Reference CPU arm for bench.py: the per-step hot path of a batch decode
// (enc Q -> shard_attention over the node's scrambled shard -> dec_output ->
// merge_shards) for `n_pairs` (request, head) pairs, each over `n_nodes`
// shards of `lk` keys, spread over `n_threads` std::threads (the reference
// functions are pure). The scrambled K'/V' shards are
// built once, outside the timed region (they are the resident KV cache).
// Runs n_steps timed steps over the same resident shards, writing each step's wall seconds to
// step_seconds[i]; returns the median.
double ref_bench_decode(std::size_t n_pairs, std::size_t n_nodes, std::size_t lk, std::size_t d,
                        std::size_t n_heads, int n_threads, int wire_fmt, int n_steps, double* step_seconds) {
    const FloatFormat wf = static_cast<FloatFormat>(wire_fmt);
    struct Pair {
        Matrix q;
        std::vector<ScramblerKeySet> ks;
        std::vector<ScrambledTriple> kv;
        Matrix out;
    };
    std::vector<Pair> pairs(n_pairs);
    // Setup (not timed): per-pair inputs from a per-pair stream, key sets, and the scrambled
    // resident shards, built in parallel.
    auto setup = [&](std::size_t p) {
        RngStream rng(derive_seed(12345, {p}));
        auto rnd = [&](std::size_t r, std::size_t c) {
            Matrix m(r, c);
            for (double& x : m.data) x = round_to_format(rng.next_gaussian(), wf);
            return m;
        };
        pairs[p].q = rnd(1, d);
        for (std::size_t n = 0; n < n_nodes; ++n) {
            ScramblerKeySet ks = negotiate_keyset(
                derive_seed(1, {p + 1, 0x7365656Bull}),
                make_spec(p + 1, 0, static_cast<std::uint32_t>(n + 1), n_heads, d, 0.125, 8.0, 0, 1, 1));
            ks.p_q = ks.span_perm(0, n_nodes * lk, 1);
            ks.p_kv = ks.span_perm(1, n * lk, lk);
            Matrix k = rnd(lk, d), v = rnd(lk, d);
            ScrambledTriple t = enc_qkv(pairs[p].q, k, v, ks, p % n_heads);
            t.k_s = round_to_format(t.k_s, wf);
            t.v_s = round_to_format(t.v_s, wf);
            pairs[p].kv.push_back(std::move(t));
            pairs[p].ks.push_back(std::move(ks));
        }
    };
    {
        std::atomic<std::size_t> nxt{0};
        std::vector<std::thread> th;
        for (int i = 0; i < n_threads; ++i)
            th.emplace_back([&] {
                for (std::size_t p; (p = nxt.fetch_add(1)) < n_pairs;) setup(p);
            });
        for (auto& t : th) t.join();
    }
    std::atomic<std::size_t> next{0};
    auto worker = [&]() {
        for (;;) {
            const std::size_t p = next.fetch_add(1);
            if (p >= n_pairs) return;
            Pair& pr = pairs[p];
            const std::size_t head = p % n_heads;
            std::vector<AttentionShard> shards;
            for (std::size_t n = 0; n < n_nodes; ++n) {
                Matrix q_s = round_to_format(
                    permute_rows_gather(apply_phi(pr.q, pr.ks[n].phi_kq[head]), pr.ks[n].p_q), wf);
                AttentionShard scr = shard_attention(q_s, pr.kv[n].k_s, pr.kv[n].v_s, AttentionMask::none(), d);
                shards.push_back(dec_output(scr.output, scr.stats, pr.ks[n], head));
            }
            pr.out = merge_shards(shards);
        }
    };
    std::vector<double> times;
    for (int step = 0; step < (n_steps > 0 ? n_steps : 1); ++step) {
        next = 0;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < n_threads; ++i) th.emplace_back(worker);
        for (auto& t : th) t.join();
        const auto t1 = std::chrono::steady_clock::now();
        times.push_back(std::chrono::duration<double>(t1 - t0).count());
        if (step_seconds) step_seconds[step] = times.back();
    }
    std::sort(times.begin(), times.end());
    return times[times.size() / 2];
}

// quant.cpp:26-67 through the reference's own quantize_affine / dequantize
int ref_quantize_affine(const double* v, std::size_t n, int bits, std::uint8_t* codes, float* scale,
                        float* zero_point) {
    try {
        const QTensor q = quantize_affine(std::span<const double>(v, n), bits);
        std::memcpy(codes, q.codes.data(), q.codes.size());
        *scale = q.scale;
        *zero_point = q.zero_point;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

void ref_dequantize(const std::uint8_t* codes, std::size_t n, int bits, float scale, float zero_point, double* out) {
    QTensor q;
    q.bits = bits;
    q.count = n;
    q.codes.assign(codes, codes + (n * static_cast<std::size_t>(bits) + 7) / 8);
    q.scale = scale;
    q.zero_point = zero_point;
    const std::vector<double> r = dequantize(q);
    std::memcpy(out, r.data(), n * sizeof(double));
}

// frame.cpp: make a tensor frame from values (payload_from_values) and encode it
int ref_encode_frame(std::uint8_t msg_type, std::uint64_t request_id, std::uint16_t layer, std::uint16_t head,
                     std::uint16_t domain, std::uint8_t dtype, const std::uint32_t* dims, std::uint32_t n_dims,
                     const double* values, std::uint8_t* out, std::uint64_t cap, std::uint64_t* out_len) {
    try {
        Frame f;
        f.msg_type = static_cast<MsgType>(msg_type);
        f.request_id = request_id;
        f.layer = layer;
        f.head = head;
        f.domain = domain;
        f.dtype = static_cast<DtypeCode>(dtype);
        f.dims.assign(dims, dims + n_dims);
        f.payload = payload_from_values(std::span<const double>(values, f.element_count()), f.dtype);
        const std::vector<std::uint8_t> b = encode_frame(f);
        *out_len = b.size();
        if (b.size() > cap) return -2;
        std::memcpy(out, b.data(), b.size());
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// frame.cpp: decode_frame + values_from_payload; returns the element count or -1 (FrameError)
long long ref_decode_frame(const std::uint8_t* bytes, std::uint64_t n, double* values, std::uint64_t cap) {
    try {
        const Frame f = decode_frame(std::span<const std::uint8_t>(bytes, n));
        const std::vector<double> v = values_from_payload(f.payload, f.element_count(), f.dtype);
        if (v.size() > cap) return -2;
        std::memcpy(values, v.data(), v.size() * sizeof(double));
        return static_cast<long long>(v.size());
    } catch (const std::exception&) {
        return -1;
    }
}

std::uint32_t ref_crc32(const std::uint8_t* bytes, std::uint64_t n) {
    return crc32(std::span<const std::uint8_t>(bytes, n));
}

}  // extern "C"
