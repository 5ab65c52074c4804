// keys.cpp -- host-side key derivation for the scrambled attention path (product code).
//
// The protocol contract (rng.hpp:8-15) requires every participant to regenerate identical
// key sets from the shared seed, so this is a bit-exact restatement of the reference's
// SplitMix64 stream, rejection sampling, Fisher-Yates and log-uniform diagonal draws, run
// on the host once per (request, layer, domain) and packed into a flat device image.
// Not a GPU kernel: Fisher-Yates with rejection sampling is inherently serial and the
// factors need the same glibc exp/log as the reference.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <vector>

#include "sdattn_b200.h"
#include "sdattn_internal.h"

namespace sda {

// rng.hpp:16-49 -- counter-based SplitMix64 stream.
class SplitMix64 {
  public:
    explicit SplitMix64(uint64_t seed) : state_(seed) {}
    static uint64_t mix(uint64_t x) {
        x ^= x >> 30;
        x *= 0xBF58476D1CE4E5B9ULL;
        x ^= x >> 27;
        x *= 0x94D049BB133111EBULL;
        return x ^ (x >> 31);
    }
    uint64_t u64() { return mix(state_ += kGamma); }
    double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }   // rng.hpp:26
    uint64_t below(uint64_t n) {                                              // rng.cpp:8-17
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        for (;;) {
            const uint64_t x = u64();
            if (x < limit) return x % n;
        }
    }
    static constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

  private:
    uint64_t state_;
};

uint64_t derive(uint64_t base, const uint64_t* tags, size_t n) {  // rng.cpp:35-39
    for (size_t i = 0; i < n; ++i) base = SplitMix64::mix(base ^ (tags[i] + SplitMix64::kGamma));
    return base;
}

// permutation.cpp:29-37
static void fisher_yates(size_t n, SplitMix64& r, uint32_t* fwd) {
    for (size_t i = 0; i < n; ++i) fwd[i] = static_cast<uint32_t>(i);
    for (size_t i = n; i-- > 1;) {
        const size_t j = static_cast<size_t>(r.below(i + 1));
        std::swap(fwd[i], fwd[j]);
    }
}

// permutation.cpp:94-106 -- magnitude draw then sign draw, interleaved per factor.
static void log_uniform_signed(size_t d, double lo, double hi, SplitMix64& r, double* f) {
    const double log_lo = std::log(lo);
    const double log_span = std::log(hi) - log_lo;
    for (size_t i = 0; i < d; ++i) {
        const double mag = std::exp(log_lo + log_span * r.unit());
        f[i] = (r.u64() & 1) ? mag : -mag;
    }
}

// scrambler.cpp:25-36 -- draw order s1, p1, p2, s2 is part of the contract.
static void draw_scrambler(size_t d, double lo, double hi, int mode, SplitMix64& r, double* s1,
                           uint32_t* p1, uint32_t* p2, double* s2) {
    log_uniform_signed(d, lo, hi, r, s1);
    fisher_yates(d, r, p1);
    fisher_yates(d, r, p2);
    if (mode == SDA_MODE_S1_ONLY) {
        for (size_t i = 0; i < d; ++i) s2[i] = 1.0;
    } else {
        log_uniform_signed(d, lo, hi, r, s2);
    }
}

// Bank-conflict-free gather order through permutation q (sdattn_internal.h, kSched*): the
// lanes x banks multigraph with an edge (l, q[l*E+e] % 32) per element is E-regular, so E
// rounds of Kuhn's augmenting-path matching each find a perfect matching of the edges left.
static void gather_schedule(size_t d, const uint32_t* q, uint8_t* sched) {
    const int E = static_cast<int>(d / 32);
    if (E < 1) return;
    std::vector<uint8_t> used(d, 0);   // element l*E+e already scheduled
    for (int k = 0; k < E; ++k) {
        int bank_of_lane[32], lane_of_bank[32], elem_of_lane[32];
        for (int i = 0; i < 32; ++i) bank_of_lane[i] = lane_of_bank[i] = elem_of_lane[i] = -1;
        for (int l = 0; l < 32; ++l) {
            bool seen[32] = {};
            std::function<bool(int)> augment = [&](int lane) -> bool {
                for (int e = 0; e < E; ++e) {
                    const size_t j = static_cast<size_t>(lane) * E + e;
                    if (used[j]) continue;
                    const int bnk = static_cast<int>(q[j] % 32);
                    if (seen[bnk]) continue;
                    seen[bnk] = true;
                    if (lane_of_bank[bnk] < 0 || augment(lane_of_bank[bnk])) {
                        lane_of_bank[bnk] = lane;
                        bank_of_lane[lane] = bnk;
                        elem_of_lane[lane] = e;
                        return true;
                    }
                }
                return false;
            };
            augment(l);   // a perfect matching exists (regular bipartite multigraph): always succeeds
        }
        for (int l = 0; l < 32; ++l) {
            const int e = elem_of_lane[l] < 0 ? 0 : elem_of_lane[l];
            sched[l * E + k] = static_cast<uint8_t>(e);
            used[static_cast<size_t>(l) * E + e] = 1;
        }
    }
}

// Packed device scrambler (SDA_SCRAMBLER_BYTES(d) bytes), see sdattn_internal.h.
static void pack_scrambler(size_t d, const double* s1, const uint32_t* p1, const uint32_t* p2,
                           const double* s2, uint8_t* dst) {
    const double rs = 1.0 / std::sqrt(static_cast<double>(d));  // fwht.cpp:24 scale
    float* f = reinterpret_cast<float*>(dst);
    uint16_t* u = reinterpret_cast<uint16_t*>(dst + 24 * d);
    for (size_t i = 0; i < d; ++i) {
        f[kInFwd * d + i] = static_cast<float>(s1[i]);
        f[kInInvT * d + i] = static_cast<float>(1.0 / s1[i]);
        f[kOutFwd * d + i] = static_cast<float>(s2[i] * rs);
        f[kOutInvT * d + i] = static_cast<float>(rs / s2[i]);
        f[kInvIn * d + i] = static_cast<float>(1.0 / s2[i]);
        f[kInvOut * d + i] = static_cast<float>(rs / s1[i]);
        u[kP1 * d + i] = static_cast<uint16_t>(p1[i]);
        u[kP2 * d + i] = static_cast<uint16_t>(p2[i]);
        u[kP1Inv * d + p1[i]] = static_cast<uint16_t>(i);
        u[kP2Inv * d + p2[i]] = static_cast<uint16_t>(i);
    }
    uint8_t* sch = dst + kSchedOff * d;
    std::fill(sch, sch + 2 * d, uint8_t{0});
    gather_schedule(d, p2, sch + kSchedP2 * d);
    gather_schedule(d, p1, sch + kSchedP1 * d);
}

// FP64 mode scrambler (SDA_SCRAMBLER_BYTES_F64(d) bytes): f64 [2][d] = {s1, s2}, then the u16
// tables of pack_scrambler -- the raw factors, so the device repeats the reference's f64 ops
static void pack_scrambler_f64(size_t d, const double* s1, const uint32_t* p1, const uint32_t* p2,
                               const double* s2, uint8_t* dst) {
    double* f = reinterpret_cast<double*>(dst);
    uint16_t* u = reinterpret_cast<uint16_t*>(dst + 16 * d);
    for (size_t i = 0; i < d; ++i) {
        f[i] = s1[i];
        f[d + i] = s2[i];
        u[kP1 * d + i] = static_cast<uint16_t>(p1[i]);
        u[kP2 * d + i] = static_cast<uint16_t>(p2[i]);
        u[kP1Inv * d + p1[i]] = static_cast<uint16_t>(i);
        u[kP2Inv * d + p2[i]] = static_cast<uint16_t>(i);
    }
}

static bool pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }

}  // namespace sda

extern "C" {

uint64_t sda_derive_seed(uint64_t base, const uint64_t* tags, size_t n_tags) {
    return sda::derive(base, tags, n_tags);
}

uint64_t sda_shared_seed(uint64_t master_seed, uint64_t request_id) {
    const uint64_t tags[2] = {request_id, 0x7365656BULL};
    return sda::derive(master_seed, tags, 2);
}

sda_status sda_random_permutation(size_t n, uint64_t seed, uint32_t* forward) {
    if (n == 0 || !forward) return SDA_ERR_INVALID_ARGUMENT;  // permutation.cpp:30
    sda::SplitMix64 r(seed);
    sda::fisher_yates(n, r, forward);
    return SDA_OK;
}

sda_status sda_negotiate_keyset(uint64_t shared_seed, const sda_keyspec* spec, sda_host_keyset* out) {
    if (!spec || !out) return SDA_ERR_INVALID_ARGUMENT;
    if (!sda::pow2(spec->head_dim)) return SDA_ERR_NOT_POW2;                       // scrambler.cpp:27
    if (!(spec->mag_lo > 0.0) || !(spec->mag_hi >= spec->mag_lo)) return SDA_ERR_INVALID_ARGUMENT;  // permutation.cpp:95
    const size_t d = spec->head_dim;
    for (uint32_t h = 0; h < spec->n_heads; ++h) {   // scrambler.cpp:113-118
        const uint64_t tq[5] = {spec->request_id, spec->layer, spec->domain, 1, h};
        sda::SplitMix64 rq(sda::derive(shared_seed, tq, 5));
        sda::draw_scrambler(d, spec->mag_lo, spec->mag_hi, spec->mode, rq, out->kq_s1 + h * d,
                            out->kq_p1 + h * d, out->kq_p2 + h * d, out->kq_s2 + h * d);
        const uint64_t tv[5] = {spec->request_id, spec->layer, spec->domain, 2, h};
        sda::SplitMix64 rv(sda::derive(shared_seed, tv, 5));
        sda::draw_scrambler(d, spec->mag_lo, spec->mag_hi, spec->mode, rv, out->v_s1 + h * d,
                            out->v_p1 + h * d, out->v_p2 + h * d, out->v_s2 + h * d);
    }
    const uint64_t tt[5] = {spec->request_id, spec->layer, spec->domain, 3, 0};     // scrambler.cpp:119-120
    out->token_perm_seed = sda::derive(shared_seed, tt, 5);
    return SDA_OK;
}

sda_status sda_span_perm(uint64_t token_perm_seed, uint64_t tag, uint64_t first_pos, size_t len,
                         uint32_t* forward) {
    if (len == 0 || !forward) return SDA_ERR_INVALID_ARGUMENT;  // negotiate_keyset: lengths >= 1
    const uint64_t tags[3] = {tag, first_pos, static_cast<uint64_t>(len)};
    sda::SplitMix64 r(sda::derive(token_perm_seed, tags, 3));
    sda::fisher_yates(len, r, forward);
    return SDA_OK;
}

sda_status sda_invert_permutation(const uint32_t* forward, size_t n, uint32_t* inverse) {
    if (!forward || !inverse) return SDA_ERR_INVALID_ARGUMENT;
    std::vector<uint8_t> seen(n, 0);
    for (size_t i = 0; i < n; ++i) {
        if (forward[i] >= n || seen[forward[i]]) return SDA_ERR_INVALID_ARGUMENT;
        seen[forward[i]] = 1;
        inverse[forward[i]] = static_cast<uint32_t>(i);
    }
    return SDA_OK;
}

size_t sda_keyset_bytes(uint32_t n_heads, uint32_t head_dim) {
    return static_cast<size_t>(n_heads) * SDA_KEYSET_HEAD_BYTES(head_dim);
}

sda_status sda_pack_keyset(const sda_host_keyset* ks, uint32_t n_heads, uint32_t head_dim, void* out) {
    if (!ks || !out) return SDA_ERR_INVALID_ARGUMENT;
    if (!sda::pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (head_dim > 65536) return SDA_ERR_UNSUPPORTED;
    const size_t d = head_dim;
    uint8_t* dst = static_cast<uint8_t*>(out);
    for (uint32_t h = 0; h < n_heads; ++h) {
        uint8_t* head = dst + h * SDA_KEYSET_HEAD_BYTES(d);
        sda::pack_scrambler(d, ks->kq_s1 + h * d, ks->kq_p1 + h * d, ks->kq_p2 + h * d, ks->kq_s2 + h * d, head);
        sda::pack_scrambler(d, ks->v_s1 + h * d, ks->v_p1 + h * d, ks->v_p2 + h * d, ks->v_s2 + h * d,
                            head + SDA_SCRAMBLER_BYTES(d));
    }
    return SDA_OK;
}

size_t sda_keyset_bytes_f64(uint32_t n_heads, uint32_t head_dim) {
    return static_cast<size_t>(n_heads) * SDA_KEYSET_HEAD_BYTES_F64(head_dim);
}

sda_status sda_pack_keyset_f64(const sda_host_keyset* ks, uint32_t n_heads, uint32_t head_dim, void* out) {
    if (!ks || !out) return SDA_ERR_INVALID_ARGUMENT;
    if (!sda::pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (head_dim > 65536) return SDA_ERR_UNSUPPORTED;
    const size_t d = head_dim;
    uint8_t* dst = static_cast<uint8_t*>(out);
    for (uint32_t h = 0; h < n_heads; ++h) {
        uint8_t* head = dst + h * SDA_KEYSET_HEAD_BYTES_F64(d);
        sda::pack_scrambler_f64(d, ks->kq_s1 + h * d, ks->kq_p1 + h * d, ks->kq_p2 + h * d, ks->kq_s2 + h * d, head);
        sda::pack_scrambler_f64(d, ks->v_s1 + h * d, ks->v_p1 + h * d, ks->v_p2 + h * d, ks->v_s2 + h * d,
                                head + SDA_SCRAMBLER_BYTES_F64(d));
    }
    return SDA_OK;
}

}  // extern "C"
