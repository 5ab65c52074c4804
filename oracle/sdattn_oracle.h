/*
 * sdattn_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, f64) of the reference's scrambled-distributed-
 * attention hot path (/root/reference/proj/core). It is the parity checker
 * for the CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product library
 * (paper_2605_25716_b200/libsdattn_b200.so) never links or calls it.
 *
 * Parity of this restatement is pinned two ways:
 *   1. against the reference itself, compiled from its own sources into
 *      oracle/_ref/libsdattn_ref.so by oracle/Makefile (tests/test_oracle_ref.py),
 *   2. against golden vectors generated from that build and committed under
 *      tests/golden/ (tests/golden/make_golden.py), plus the reference's own
 *      known-answer tests (test_tensor.cpp:94-100).
 */
#ifndef SDATTN_ORACLE_H
#define SDATTN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng (rng.hpp:16-53, rng.cpp:8-39) -------------------------------- */
typedef struct {
    uint64_t state;
    int have_cached;
    double cached;
} or_rng;

void or_rng_init(or_rng* r, uint64_t seed);
uint64_t or_mix(uint64_t x);
uint64_t or_next_u64(or_rng* r);
double or_next_double(or_rng* r);
uint64_t or_next_below(or_rng* r, uint64_t n);
double or_next_gaussian(or_rng* r);
uint64_t or_derive_seed(uint64_t base, const uint64_t* tags, size_t n_tags);
/* n gaussians from a fresh stream seeded with `seed` */
void or_gaussian_fill(uint64_t seed, size_t n, double* out);

/* ---- permutation / diag scaling (permutation.cpp:29-106) -------------- */
/* forward[i] = where index i lands; returns 0 or -1 on n == 0 */
int or_random_permutation(size_t n, or_rng* r, uint32_t* forward);
int or_random_diag_scaling(size_t d, double lo, double hi, or_rng* r, double* factors);

/* ---- fwht (fwht.cpp:10-26) -------------------------------------------- */
int or_fwht_normalized_inplace(double* x, size_t n);

/* ---- float formats (float_format.cpp:26-58) ---------------------------- */
enum { OR_FMT_F64 = 0, OR_FMT_F32 = 1, OR_FMT_BF16 = 2, OR_FMT_F16 = 3 };
double or_round_to_format(double x, int fmt);
void or_round_array(double* x, size_t n, int fmt);

/* ---- scrambler (scrambler.hpp:21-36, scrambler.cpp:25-124) ------------- */
enum { OR_MODE_S1_AND_S2 = 0, OR_MODE_S1_ONLY = 1 };
enum { OR_PHI_FORWARD = 0, OR_PHI_INV_T = 1, OR_PHI_INV = 2 };

/* One structured scrambler phi = S1 P1 H P2 S2 over dimension d. Buffers are
 * caller-owned, each of length d. */
typedef struct {
    size_t dim;
    double* s1;
    uint32_t* p1;
    uint32_t* p2;
    double* s2;
    int with_hadamard;
} or_scrambler;

int or_build_scrambler(size_t d, double lo, double hi, or_rng* r, int mode, or_scrambler* out);
/* x: rows x d row-major; out may not alias x. */
int or_apply_phi(const double* x, size_t rows, const or_scrambler* s, int variant, double* out);

/* Key-set derivation (scrambler.cpp:99-124). Flat layout:
 *   kq_s1/kq_s2/v_s1/v_s2: [n_heads][d] f64, kq_p1/...: [n_heads][d] u32.  */
typedef struct {
    uint64_t request_id;
    uint32_t layer;
    uint32_t domain;
    size_t n_heads;
    size_t head_dim;
    double mag_lo;
    double mag_hi;
    int mode;
} or_keyspec;

typedef struct {
    double* kq_s1; uint32_t* kq_p1; uint32_t* kq_p2; double* kq_s2;
    double* v_s1;  uint32_t* v_p1;  uint32_t* v_p2;  double* v_s2;
    uint64_t token_perm_seed;
} or_keyset;

int or_negotiate_keyset(uint64_t shared_seed, const or_keyspec* spec, or_keyset* out);
int or_span_perm(uint64_t token_perm_seed, uint64_t tag, uint64_t first_pos, size_t len,
                 uint32_t* forward);
/* View head h of a keyset as a scrambler (which = 0: phi_kq, 1: phi_v). */
void or_keyset_head(const or_keyset* ks, size_t d, size_t head, int which, or_scrambler* out);

/* ---- attention (attention.cpp:42-123) ---------------------------------- */
enum { OR_MASK_NONE = 0, OR_MASK_CAUSAL = 1 };
/* q: lq x d, k/v: lk x d. out: lq x d, row_max/exp_sum: lq.
 * Returns 0, or -1 on bad shapes. */
int or_shard_attention(const double* q, size_t lq, const double* k, const double* v, size_t lk,
                       size_t d, int mask_kind, int64_t causal_offset, double* out,
                       double* row_max, double* exp_sum);
/* n shards, each: out_i (rows x cols), row_max_i, exp_sum_i given as arrays
 * of pointers. Returns 0, -1 (empty list), -2 (row masked everywhere). */
int or_merge_shards(size_t n, const double* const* outs, const double* const* row_max,
                    const double* const* exp_sum, size_t rows, size_t cols, double* merged);

/* ---- enc / dec (scrambler.cpp:126-149) --------------------------------- */
/* gather rows: out[i] = m[p[i]] ; scatter rows: out[p[i]] = m[i] */
void or_permute_rows_gather(const double* m, size_t rows, size_t cols, const uint32_t* p,
                            double* out);
void or_permute_rows_scatter(const double* m, size_t rows, size_t cols, const uint32_t* p,
                             double* out);
int or_enc_rows(const double* x, size_t rows, const or_scrambler* s, int variant,
                const uint32_t* perm, double* out);
int or_dec_output(const double* o_s, const double* row_max_s, const double* exp_sum_s,
                  size_t lq, const or_scrambler* phi_v, const uint32_t* p_q, double* out,
                  double* row_max, double* exp_sum);

/* quant.cpp:26-67 */
int or_quantize_affine(const double* v, size_t n, int bits, uint8_t* codes, float* scale, float* zero_point);
void or_dequantize(const uint8_t* codes, size_t n, int bits, float scale, float zero_point, double* out);

/* frame.cpp:78-83 */
uint32_t or_crc32(const uint8_t* b, size_t n);

#ifdef __cplusplus
}
#endif
#endif
