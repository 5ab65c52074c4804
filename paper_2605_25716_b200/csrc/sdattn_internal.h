// sdattn_internal.h -- layouts shared by the host packer and the sm_100a kernels.
#pragma once
#include <cstddef>
#include <cstdint>

#include "sdattn_b200.h"

namespace sda {

constexpr int kMaxPeers = 16;

// Packed device scrambler for head dim d (SDA_SCRAMBLER_BYTES(d) = 34 d bytes):
//   f32 tables [6][d], u16 tables [4][d], then u8 gather schedules [2][d] (d >= 32; zero below):
//   a warp that owns elements [lane*E, lane*E+E) (E = d/32) and gathers them through a permutation
//   Q from a row in shared memory issues E loads; in load k lane l takes its element
//   e = sched[l*E + k], chosen so that the 32 addresses Q[l*E + e] of every load fall in 32
//   different banks. Q's values mod 32 put exactly E of a lane's and E of a bank's elements on each
//   side of a lanes x banks multigraph that is E-regular, so it splits into E perfect matchings
//   (Konig) -- one per load. kSchedP2: the gather u[j] = t[P2[j]]; kSchedP1: y[i] = w[P1[i]].
// With R = 1/sqrt(d) (the normalised FWHT scale, fwht.cpp:24) and the raw +-1 butterfly H:
//   x phi      : y[k] = OutFwd[k]  * H(u)[P2Inv[k]],  u[P1[i]] = x[i] * InFwd[i]
//   x phi^{-T} : y[k] = OutInvT[k] * H(u)[P2Inv[k]],  u[P1[i]] = x[i] * InInvT[i]
//   x phi^{-1} : y[i] = InvOut[i]  * H(u)[P1[i]],     u[j]     = x[P2[j]] * InvIn[P2[j]]
// (scrambler.cpp:42-63 with the componentwise steps folded into gathers / scatters.)
enum : int { kInFwd = 0, kInInvT = 1, kOutFwd = 2, kOutInvT = 3, kInvIn = 4, kInvOut = 5 };
enum : int { kP1 = 0, kP2 = 1, kP1Inv = 2, kP2Inv = 3 };
enum : int { kSchedP2 = 0, kSchedP1 = 1 };
constexpr int kU16Off = 24;   // u16 tables at 24 d bytes
constexpr int kSchedOff = 32; // u8 schedules at 32 d bytes

uint64_t derive(uint64_t base, const uint64_t* tags, size_t n);
void count_launch();   // sda_launch_count() bookkeeping for kernels launched outside capi.cu

// Kernel parameter blocks (passed by value to the kernels).
struct K1Params {
    const void* x;
    void* out;
    const void* keys;
    const uint32_t* perm;
    int64_t keys_bstride;
    int64_t perm_bstride;
    int64_t rows;
    int64_t out_rows_cap;
    int64_t out_row_offset;
    int n_heads;
    int key_heads;
    int which;    // 0 phi_kq, 1 phi_v
    int inv_t;    // 1: phi^{-T}
    int64_t x_batch_mod;   // > 0: request b reads x[b % x_batch_mod] (one Q, many key sets)
    // LL exchange (decode, rows == 1; epoch != nullptr): request b's Q' row goes to
    // ll_out[b / x_batch_mod] (a peer's receive slot, [x_batch_mod][n_heads][d] in LL format:
    // every 4-byte data word is followed by the 4-byte step epoch, see ll_store)
    void* ll_out[kMaxPeers];
    const uint32_t* epoch;
    // quantised wire in the epilogue (sda_scramble_quant): out = dequantize(quantize_affine(.))
    // per (request, head) tensor, from the per-tensor min / max keys of a first pass
    int quant_bits;
    unsigned long long* qscratch;   // [2][n_batch * n_heads] order-preserving min / max keys
    int32_t* qerr;
};

struct K2Params {
    const void* q;
    const void* k;
    const void* v;
    const int32_t* kv_len;
    float* out_o;
    float* out_stats;
    int64_t kv_cap;
    int64_t n_batch;
    int64_t q_rows;
    int q_heads;
    int kv_heads;
    int n_splits;
    float scale;   // 1/sqrt(d) (attention.cpp:45)
    int causal;            // 1: key j visible to query row i iff j <= i + causal_offset (attention.hpp:25-27)
    int64_t causal_offset;
    // LL exchange (decode, q_rows == 1; epoch != nullptr): q is in LL format (spin until its
    // words carry *epoch); split `split` of request b = (dest, i) = (b / b_per, b % b_per) is
    // written as an LL record row [d O' | row_max, exp_sum] at logical float
    // ((split * b_per + i) * q_heads + h) * (d + 2) of ll_rec[dest] (8 bytes per float)
    const uint32_t* epoch;
    int64_t b_per;
    void* ll_rec[kMaxPeers];
    // remote records (prefill, one split): request b = (dest, i) writes its packed record
    // [q_heads * q_rows * d O' | q_heads * q_rows * 2 stats] straight into ll_rec[dest] +
    // i * rec_stride floats (a peer's receive slot, plain stores); the CTA completing a
    // destination raises *peer_flag[dest] = *epoch (system-scope release)
    int remote_rec;
    int64_t rec_stride;
    uint32_t* peer_flag[kMaxPeers];
    uint32_t* dest_counters;   // [n_dest] zeroed, self-resetting
    // stream-K workspace of the tensor-core prefill form (one split): caller-owned, zeroed once,
    // left zeroed by every launch; null -> split grid
    void* sk_work;
    size_t sk_work_bytes;
};

struct K3Source {
    const float* o;
    const float* stats;
    const uint8_t* keys;
    const uint32_t* pq_inv;
    int64_t bstride;       // elements between requests (o and stats); 0 = dense
};

struct K3Params {
    K3Source src[SDA_MAX_SOURCES];
    int n_src;
    int64_t keys_bstride;
    int key_heads;
    int64_t pq_bstride;
    int64_t n_batch;
    int q_heads;
    int64_t q_rows;
    void* out;
    float* out_stats;
    int32_t* err;
    int64_t out_bstride;   // elements between requests (out and out_stats); 0 = dense
    // LL exchange: sources are LL record rows (src.o = byte base, row (b, h) at logical float
    // b * bstride + h * (d + 2), stats at + d; q_rows == 1), read by spinning until they carry
    // *epoch; the last CTA then bumps *epoch (done_counter: one zeroed u32, self-resetting)
    int ll;
    uint32_t* epoch;
    uint32_t* done_counter;
    // quantised O' wire (sda_unscramble_merge_quant): every key group's O' quantised + dequantised
    // before its unscramble; qpass 1 = the min / max pass over (group, request, head) tensors
    int quant_bits;
    int qpass;
    int n_groups;
    unsigned long long* qscratch;   // [2][n_groups][n_batch * q_heads] min / max keys
};

}  // namespace sda

#include <cuda_runtime.h>
namespace sda {
cudaError_t launch_k1(const K1Params& p, int d, int xdt, int odt, int64_t n_batch, cudaStream_t st);
// K3 on the tensor cores (k3_tc.cu); cudaErrorNotSupported when the merge is not eligible
cudaError_t launch_k3_tc(const K3Params& p, int d, int odt, cudaStream_t st);
bool k1_tc_eligible(const K1Params& p, int d, int xdt, int odt);
cudaError_t launch_k1_tc(const K1Params& p, int d, int64_t n_batch, cudaStream_t st);
cudaError_t launch_quantize(const void* x, int dt, int64_t n, int64_t count, int bits, uint8_t* codes,
                            int64_t codes_stride, float* scale, float* zero, unsigned long long* scratch, int32_t* err,
                            cudaStream_t st);
cudaError_t launch_dequantize(const uint8_t* codes, int64_t codes_stride, const float* scale, const float* zero,
                              int64_t n, int64_t count, int bits, void* out, int dt, cudaStream_t st);
uint64_t crc_scratch_words(uint64_t len);
int k2_decode_ctas_per_sm();
cudaError_t launch_ll_unpack_q(const void* ll_q, int64_t elems, void* out, const uint32_t* epoch, cudaStream_t st);
cudaError_t launch_crc32(const uint8_t* msg, uint64_t len, uint32_t* scratch, uint8_t* out4, cudaStream_t st);
cudaError_t launch_frame_encode(const void* x, int x_dt, int64_t count, int wire, const uint8_t* header, int hlen,
                                uint8_t* out, uint64_t payload_bytes, uint32_t* crc_scratch, uint64_t* q_scratch,
                                float* q_sz, int32_t* err, cudaStream_t st);
cudaError_t launch_frame_decode(const uint8_t* frame, int hlen, uint64_t payload_bytes, int64_t count, int wire,
                                void* out, int out_dt, uint32_t* crc_scratch, float* q_sz, int32_t* err,
                                cudaStream_t st);
cudaError_t launch_wire_round(void* x, int dt, int64_t n, int fmt, cudaStream_t st);
cudaError_t launch_quant_roundtrip(void* x, int dt, int64_t n, int64_t count, int bits, unsigned long long* scratch,
                                   int32_t* err, cudaStream_t st);
cudaError_t launch_k1_tc_multi(const K1Params* p, const int64_t* n_batch, int n_jobs, int d, cudaStream_t st,
                               uint32_t* const* peer_flag = nullptr, const uint32_t* epoch = nullptr,
                               uint32_t* counters = nullptr);
cudaError_t launch_k2_decode(const K2Params& p, int d, int qdt, int kvdt, cudaStream_t st);
bool k2_prefill_tc_eligible(const K2Params& p, int d, int qdt, int kvdt);
cudaError_t launch_k2_prefill_tc(const K2Params& p, cudaStream_t st);
// bytes of the stream-K workspace for this shape (one split), 0 when it does not run stream-K
size_t k2_prefill_sk_workspace_bytes(const K2Params& p);
bool k2_gqa_tc_eligible(const K2Params& p, int d, int qdt, int kvdt);
cudaError_t launch_k2_gqa_tc(const K2Params& p, cudaStream_t st);
cudaError_t launch_k3(const K3Params& p, int d, int odt, cudaStream_t st);
cudaError_t launch_project_scramble(const void* x, int64_t n_batch, int64_t x_rows, int d_model, const void* w,
                                    int n_heads, int d, const void* keys, int64_t keys_bstride, int key_heads,
                                    int variant, int which, const uint32_t* perm, int64_t perm_bstride, int64_t rows,
                                    void* out, int64_t out_rows_cap, int64_t out_row_offset, cudaStream_t st);
// FP64 mode (f64_path.cu): which 1 = K1 (K1Params), 2 = K2 (K2Params), 3 = K3 (K3Params)
cudaError_t launch_f64_path(int which, const void* params, int d, int64_t n_batch, cudaStream_t st);
// per-TU spin budget / error word (common.cuh SDA_SPIN_ACCESSOR)
cudaError_t spin_access_exchange(const unsigned long long* set, int* err, int clear);
cudaError_t spin_access_k2_decode(const unsigned long long* set, int* err, int clear);
cudaError_t spin_access_k3_merge(const unsigned long long* set, int* err, int clear);

}  // namespace sda
