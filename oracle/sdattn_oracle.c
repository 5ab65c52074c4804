/*
 * sdattn_oracle.c -- TEST INFRASTRUCTURE ONLY (see sdattn_oracle.h).
 *
 * A plain-C, f64 restatement of the reference hot path. Every function cites
 * the reference file:line it restates (paths relative to
 * /root/reference/proj/core/). Bit-exactness with the reference relies on the
 * same IEEE-754 double arithmetic and the same glibc libm (exp, log, sqrt,
 * sin, cos, nearbyint), which the GPU box shares with this container.
 */
#define _GNU_SOURCE
#include "sdattn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN_GAMMA 0x9E3779B97F4A7C15ULL

/* rng.hpp:18 */
void or_rng_init(or_rng* r, uint64_t seed) {
    r->state = seed;
    r->have_cached = 0;
    r->cached = 0.0;
}

/* rng.hpp:36-43 -- SplitMix64 finaliser */
uint64_t or_mix(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return x;
}

/* rng.hpp:20-23 */
uint64_t or_next_u64(or_rng* r) {
    r->state += GOLDEN_GAMMA;
    return or_mix(r->state);
}

/* rng.hpp:26 -- 53 random bits scaled by 2^-53 */
double or_next_double(or_rng* r) { return (double)(or_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.cpp:8-17 -- rejection sampling below the largest multiple of n */
uint64_t or_next_below(or_rng* r, uint64_t n) {
    if (n == 0) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = or_next_u64(r);
    } while (x >= limit);
    return x % n;
}

/* rng.cpp:19-33 -- Box-Muller with one cached value, u clamped at 2^-60 */
double or_next_gaussian(or_rng* r) {
    if (r->have_cached) {
        r->have_cached = 0;
        return r->cached;
    }
    double u = or_next_double(r);
    double v = or_next_double(r);
    if (u < 0x1.0p-60) u = 0x1.0p-60;
    const double rad = sqrt(-2.0 * log(u));
    const double t = 2.0 * M_PI * v;
    r->cached = rad * sin(t);
    r->have_cached = 1;
    return rad * cos(t);
}

/* rng.cpp:35-39 -- fold each tag through the mixer */
uint64_t or_derive_seed(uint64_t base, const uint64_t* tags, size_t n_tags) {
    uint64_t s = base;
    for (size_t i = 0; i < n_tags; ++i) s = or_mix(s ^ (tags[i] + GOLDEN_GAMMA));
    return s;
}

void or_gaussian_fill(uint64_t seed, size_t n, double* out) {
    or_rng r;
    or_rng_init(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = or_next_gaussian(&r);
}

/* permutation.cpp:29-37 -- Fisher-Yates from the top, j = next_below(i+1) */
int or_random_permutation(size_t n, or_rng* r, uint32_t* fwd) {
    if (n == 0) return -1;
    for (size_t i = 0; i < n; ++i) fwd[i] = (uint32_t)i;
    for (size_t i = n - 1; i > 0; --i) {
        const size_t j = (size_t)or_next_below(r, (uint64_t)i + 1);
        const uint32_t t = fwd[i];
        fwd[i] = fwd[j];
        fwd[j] = t;
    }
    return 0;
}

/* permutation.cpp:94-106 -- interleaved draws: magnitude, then sign bit */
int or_random_diag_scaling(size_t d, double lo, double hi, or_rng* r, double* f) {
    if (!(lo > 0.0) || !(hi >= lo)) return -1;
    const double log_lo = log(lo);
    const double log_span = log(hi) - log_lo;
    for (size_t i = 0; i < d; ++i) {
        const double mag = exp(log_lo + log_span * or_next_double(r));
        const double sign = (or_next_u64(r) & 1) ? 1.0 : -1.0;
        f[i] = sign * mag;
    }
    return 0;
}

static int is_pow2(size_t n) { return n != 0 && (n & (n - 1)) == 0; }

/* fwht.cpp:10-26 -- butterflies half = 1, 2, 4, ..., then one 1/sqrt(n) scale */
int or_fwht_normalized_inplace(double* x, size_t n) {
    if (!is_pow2(n)) return -1;
    for (size_t half = 1; half < n; half <<= 1)
        for (size_t base = 0; base < n; base += half << 1)
            for (size_t i = base; i < base + half; ++i) {
                const double a = x[i], b = x[i + half];
                x[i] = a + b;
                x[i + half] = a - b;
            }
    const double scale = 1.0 / sqrt((double)n);
    for (size_t i = 0; i < n; ++i) x[i] *= scale;
    return 0;
}

/* float_format.cpp:26-35 -- single RNE rounding of a double onto a grid with
 * `mant` explicit bits and minimum normal exponent `emin`, overflow clamps. */
static double round_spec(double x, int mant, int emin, double max_finite) {
    if (x == 0.0 || isnan(x)) return x;
    if (isinf(x)) return copysign(max_finite, x);
    const int e = ilogb(x);
    const int q = (e < emin ? emin : e) - mant;
    const double quantum = ldexp(1.0, q);
    double y = nearbyint(x / quantum) * quantum;
    if (fabs(y) > max_finite) y = copysign(max_finite, y);
    return y;
}

/* float_format.cpp:39-51 */
double or_round_to_format(double x, int fmt) {
    switch (fmt) {
        case OR_FMT_F64: return x;
        case OR_FMT_F32: return (double)(float)x;
        case OR_FMT_BF16: return round_spec(x, 7, -126, 0x1.FEp127);
        case OR_FMT_F16: return round_spec(x, 10, -14, 65504.0);
        default: return x;
    }
}

/* float_format.cpp:53-58 */
void or_round_array(double* x, size_t n, int fmt) {
    if (fmt == OR_FMT_F64) return;
    for (size_t i = 0; i < n; ++i) x[i] = or_round_to_format(x[i], fmt);
}

/* scrambler.cpp:25-36 -- draw order s1, p1, p2, s2 (s1_only: s2 = 1, no draw) */
int or_build_scrambler(size_t d, double lo, double hi, or_rng* r, int mode, or_scrambler* out) {
    if (!is_pow2(d)) return -1;
    out->dim = d;
    out->with_hadamard = 1;
    if (or_random_diag_scaling(d, lo, hi, r, out->s1)) return -1;
    or_random_permutation(d, r, out->p1);
    or_random_permutation(d, r, out->p2);
    if (mode == OR_MODE_S1_ONLY) {
        for (size_t i = 0; i < d; ++i) out->s2[i] = 1.0;
    } else if (or_random_diag_scaling(d, lo, hi, r, out->s2)) {
        return -1;
    }
    return 0;
}

/* scrambler.cpp:42-63 -- one row through phi / phi^{-T} / phi^{-1}.
 *   forward: x S1 -> scatter P1 -> H -> scatter P2 -> S2
 *   inv_t  : x / S1 -> scatter P1 -> H -> scatter P2 -> / S2
 *   inv    : x / S2 -> gather P2 -> H -> gather P1 -> / S1            */
static void apply_row(const double* in, double* out, double* tmp, const or_scrambler* s,
                      int variant) {
    const size_t d = s->dim;
    if (variant == OR_PHI_INV) {
        for (size_t i = 0; i < d; ++i) tmp[i] = in[i] / s->s2[i];
        for (size_t i = 0; i < d; ++i) out[i] = tmp[s->p2[i]];
        if (s->with_hadamard) or_fwht_normalized_inplace(out, d);
        for (size_t i = 0; i < d; ++i) tmp[i] = out[s->p1[i]];
        for (size_t i = 0; i < d; ++i) out[i] = tmp[i] / s->s1[i];
        return;
    }
    const int inv = variant == OR_PHI_INV_T;
    for (size_t i = 0; i < d; ++i) tmp[i] = inv ? in[i] / s->s1[i] : in[i] * s->s1[i];
    for (size_t i = 0; i < d; ++i) out[s->p1[i]] = tmp[i];
    if (s->with_hadamard) or_fwht_normalized_inplace(out, d);
    for (size_t i = 0; i < d; ++i) tmp[s->p2[i]] = out[i];
    for (size_t i = 0; i < d; ++i) out[i] = inv ? tmp[i] / s->s2[i] : tmp[i] * s->s2[i];
}

/* scrambler.cpp:65-85 */
int or_apply_phi(const double* x, size_t rows, const or_scrambler* s, int variant, double* out) {
    double* tmp = (double*)malloc(sizeof(double) * s->dim);
    if (!tmp) return -1;
    for (size_t r = 0; r < rows; ++r)
        apply_row(x + r * s->dim, out + r * s->dim, tmp, s, variant);
    free(tmp);
    return 0;
}

/* scrambler.cpp:99-103 -- span_perm(tag, first_pos, len) */
int or_span_perm(uint64_t token_perm_seed, uint64_t tag, uint64_t first_pos, size_t len,
                 uint32_t* fwd) {
    const uint64_t tags[3] = {tag, first_pos, (uint64_t)len};
    or_rng r;
    or_rng_init(&r, or_derive_seed(token_perm_seed, tags, 3));
    return or_random_permutation(len, &r, fwd);
}

/* scrambler.cpp:105-124 -- per head h: phi_kq from tag 1, phi_v from tag 2;
 * token_perm_seed from tag 3, head 0. (p_q / p_kv are span_perms the caller
 * derives as needed.) */
int or_negotiate_keyset(uint64_t shared_seed, const or_keyspec* spec, or_keyset* out) {
    const size_t d = spec->head_dim;
    for (size_t h = 0; h < spec->n_heads; ++h) {
        or_scrambler s;
        or_rng r;
        const uint64_t tq[5] = {spec->request_id, spec->layer, spec->domain, 1, (uint64_t)h};
        or_rng_init(&r, or_derive_seed(shared_seed, tq, 5));
        s.s1 = out->kq_s1 + h * d; s.p1 = out->kq_p1 + h * d;
        s.p2 = out->kq_p2 + h * d; s.s2 = out->kq_s2 + h * d;
        if (or_build_scrambler(d, spec->mag_lo, spec->mag_hi, &r, spec->mode, &s)) return -1;
        const uint64_t tv[5] = {spec->request_id, spec->layer, spec->domain, 2, (uint64_t)h};
        or_rng_init(&r, or_derive_seed(shared_seed, tv, 5));
        s.s1 = out->v_s1 + h * d; s.p1 = out->v_p1 + h * d;
        s.p2 = out->v_p2 + h * d; s.s2 = out->v_s2 + h * d;
        if (or_build_scrambler(d, spec->mag_lo, spec->mag_hi, &r, spec->mode, &s)) return -1;
    }
    const uint64_t tt[5] = {spec->request_id, spec->layer, spec->domain, 3, 0};
    out->token_perm_seed = or_derive_seed(shared_seed, tt, 5);
    return 0;
}

void or_keyset_head(const or_keyset* ks, size_t d, size_t h, int which, or_scrambler* s) {
    s->dim = d;
    s->with_hadamard = 1;
    if (which == 0) {
        s->s1 = ks->kq_s1 + h * d; s->p1 = ks->kq_p1 + h * d;
        s->p2 = ks->kq_p2 + h * d; s->s2 = ks->kq_s2 + h * d;
    } else {
        s->s1 = ks->v_s1 + h * d; s->p1 = ks->v_p1 + h * d;
        s->p2 = ks->v_p2 + h * d; s->s2 = ks->v_s2 + h * d;
    }
}

/* attention.cpp:42-78 -- two-pass softmax per row: max of scaled logits,
 * then exp-sum and the weighted V accumulation, normalised at the end. A
 * fully masked row keeps row_max = -inf, exp_sum = 0, output 0. */
int or_shard_attention(const double* q, size_t lq, const double* k, const double* v, size_t lk,
                       size_t d, int mask_kind, int64_t causal_offset, double* out,
                       double* row_max, double* exp_sum) {
    const double scale = 1.0 / sqrt((double)d);
    double* logits = (double*)malloc(sizeof(double) * (lk ? lk : 1));
    if (!logits) return -1;
    for (size_t i = 0; i < lq; ++i) {
        const double* qi = q + i * d;
        double* orow = out + i * d;
        for (size_t c = 0; c < d; ++c) orow[c] = 0.0;
        double m = -INFINITY;
        for (size_t j = 0; j < lk; ++j) {
            const int ok = mask_kind == OR_MASK_NONE ||
                           (int64_t)j <= (int64_t)i + causal_offset; /* attention.cpp:16-27 */
            if (!ok) {
                logits[j] = -INFINITY;
                continue;
            }
            double dot = 0.0; /* matrix.cpp dot(): sequential sum */
            for (size_t c = 0; c < d; ++c) dot += qi[c] * k[j * d + c];
            logits[j] = dot * scale;
            if (logits[j] > m) m = logits[j];
        }
        row_max[i] = -INFINITY;
        exp_sum[i] = 0.0;
        if (!isfinite(m)) continue;
        double s = 0.0;
        for (size_t j = 0; j < lk; ++j) {
            if (logits[j] == -INFINITY) continue;
            const double w = exp(logits[j] - m);
            s += w;
            for (size_t c = 0; c < d; ++c) orow[c] += w * v[j * d + c];
        }
        for (size_t c = 0; c < d; ++c) orow[c] /= s;
        row_max[i] = m;
        exp_sum[i] = s;
    }
    free(logits);
    return 0;
}

/* attention.cpp:89-123 -- running-max merge; one shard is returned verbatim */
int or_merge_shards(size_t n, const double* const* outs, const double* const* rmax,
                    const double* const* esum, size_t rows, size_t cols, double* merged) {
    if (n == 0) return -1;
    if (n == 1) {
        for (size_t i = 0; i < rows; ++i)
            if (esum[0][i] == 0.0) return -2;
        memcpy(merged, outs[0], sizeof(double) * rows * cols);
        return 0;
    }
    for (size_t i = 0; i < rows; ++i) {
        double m_star = -INFINITY;
        for (size_t s = 0; s < n; ++s)
            if (esum[s][i] > 0.0 && rmax[s][i] > m_star) m_star = rmax[s][i];
        if (!isfinite(m_star)) return -2;
        double denom = 0.0;
        double* orow = merged + i * cols;
        for (size_t c = 0; c < cols; ++c) orow[c] = 0.0;
        for (size_t s = 0; s < n; ++s) {
            if (esum[s][i] == 0.0) continue;
            const double w = esum[s][i] * exp(rmax[s][i] - m_star);
            denom += w;
            for (size_t c = 0; c < cols; ++c) orow[c] += w * outs[s][i * cols + c];
        }
        for (size_t c = 0; c < cols; ++c) orow[c] /= denom;
    }
    return 0;
}

/* permutation.cpp:58-67 */
void or_permute_rows_gather(const double* m, size_t rows, size_t cols, const uint32_t* p,
                            double* out) {
    for (size_t i = 0; i < rows; ++i) memcpy(out + i * cols, m + (size_t)p[i] * cols, sizeof(double) * cols);
}

/* permutation.cpp:47-56 */
void or_permute_rows_scatter(const double* m, size_t rows, size_t cols, const uint32_t* p,
                             double* out) {
    for (size_t i = 0; i < rows; ++i) memcpy(out + (size_t)p[i] * cols, m + i * cols, sizeof(double) * cols);
}

/* scrambler.cpp:126-136 (one operand of enc_qkv): gather_rows(x * phi_variant, perm) */
int or_enc_rows(const double* x, size_t rows, const or_scrambler* s, int variant,
                const uint32_t* perm, double* out) {
    double* tmp = (double*)malloc(sizeof(double) * rows * s->dim + 1);
    if (!tmp) return -1;
    or_apply_phi(x, rows, s, variant, tmp);
    or_permute_rows_gather(tmp, rows, s->dim, perm, out);
    free(tmp);
    return 0;
}

/* scrambler.cpp:138-149 -- O = scatter_rows(O' phi_V^{-1}, p_q); stats scattered by p_q */
int or_dec_output(const double* o_s, const double* rmax_s, const double* esum_s, size_t lq,
                  const or_scrambler* phi_v, const uint32_t* p_q, double* out, double* rmax,
                  double* esum) {
    double* tmp = (double*)malloc(sizeof(double) * lq * phi_v->dim + 1);
    if (!tmp) return -1;
    or_apply_phi(o_s, lq, phi_v, OR_PHI_INV, tmp);
    or_permute_rows_scatter(tmp, lq, phi_v->dim, p_q, out);
    for (size_t i = 0; i < lq; ++i) {
        rmax[p_q[i]] = rmax_s[i];
        esum[p_q[i]] = esum_s[i];
    }
    free(tmp);
    return 0;
}

/* quant.cpp:26-51 -- per-tensor affine min-max quantisation, codes packed LSB-first.
 * codes: ceil(n * bits / 8) zero-initialised bytes. Returns -1 for bits outside [2, 8]
 * (quant.cpp:27) or a non-finite value (quant.cpp:35). */
int or_quantize_affine(const double* v, size_t n, int bits, uint8_t* codes, float* scale, float* zero_point) {
    if (bits < 2 || bits > 8) return -1;
    memset(codes, 0, (n * (size_t)bits + 7) / 8);
    *scale = 0.0f;
    *zero_point = 0.0f;
    if (n == 0) return 0;
    double lo = v[0], hi = v[0];
    for (size_t i = 0; i < n; ++i) {
        if (!isfinite(v[i])) return -1;
        if (v[i] < lo) lo = v[i];
        if (v[i] > hi) hi = v[i];
    }
    const uint32_t levels = (1u << bits) - 1u;
    *zero_point = (float)lo;
    *scale = (float)((hi - lo) / (double)levels);
    if (*scale == 0.0f) return 0;   /* constant tensor: all codes 0 */
    const double inv = 1.0 / (double)*scale;
    for (size_t i = 0; i < n; ++i) {
        double c = nearbyint((v[i] - (double)*zero_point) * inv);
        if (c < 0.0) c = 0.0;
        if (c > (double)levels) c = (double)levels;
        const uint32_t code = (uint32_t)c;
        uint64_t bit = (uint64_t)i * (uint64_t)bits;
        for (int b = 0; b < bits; ++b, ++bit)
            if (code & (1u << b)) codes[bit / 8] |= (uint8_t)(1u << (bit % 8));
    }
    return 0;
}

/* quant.cpp:55-61 -- value = code * scale + zero_point in f64 */
void or_dequantize(const uint8_t* codes, size_t n, int bits, float scale, float zero_point, double* out) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t code = 0;
        uint64_t bit = (uint64_t)i * (uint64_t)bits;
        for (int b = 0; b < bits; ++b, ++bit)
            if (codes[bit / 8] & (1u << (bit % 8))) code |= 1u << b;
        out[i] = (double)code * (double)scale + (double)zero_point;
    }
}

/* frame.cpp:17-25, :78-83 -- CRC-32/IEEE (reflected, poly 0xEDB88320, init and final xor ~0) */
uint32_t or_crc32(const uint8_t* b, size_t n) {
    uint32_t c = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; ++i) {
        c ^= b[i];
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    }
    return c ^ 0xFFFFFFFFu;
}
