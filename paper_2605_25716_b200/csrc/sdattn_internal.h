// sdattn_internal.h -- layouts shared by the host packer and the sm_100a kernels.
#pragma once
#include <cstddef>
#include <cstdint>

#include "sdattn_b200.h"

namespace sda {

constexpr int kMaxPeers = 16;

// Packed device scrambler for head dim d (SDA_SCRAMBLER_BYTES(d) = 32 d bytes):
//   f32 tables [6][d] then u16 tables [4][d].
// With R = 1/sqrt(d) (the normalised FWHT scale, fwht.cpp:24) and the raw +-1 butterfly H:
//   x phi      : y[k] = OutFwd[k]  * H(u)[P2Inv[k]],  u[P1[i]] = x[i] * InFwd[i]
//   x phi^{-T} : y[k] = OutInvT[k] * H(u)[P2Inv[k]],  u[P1[i]] = x[i] * InInvT[i]
//   x phi^{-1} : y[i] = InvOut[i]  * H(u)[P1[i]],     u[j]     = x[P2[j]] * InvIn[P2[j]]
// (scrambler.cpp:42-63 with the componentwise steps folded into gathers / scatters.)
enum : int { kInFwd = 0, kInInvT = 1, kOutFwd = 2, kOutInvT = 3, kInvIn = 4, kInvOut = 5 };
enum : int { kP1 = 0, kP2 = 1, kP1Inv = 2, kP2Inv = 3 };

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
    // fused peer push (exchange): request b's rows go to out_peer[b / x_batch_mod] (a peer's
    // receive slot, row layout as `out` with batch x_batch_mod); the last CTA of a destination
    // raises *peer_flag[dest] = *epoch (system-scope release)
    void* out_peer[kMaxPeers];
    uint32_t* peer_flag[kMaxPeers];
    const uint32_t* epoch;
    uint32_t* dest_counters;   // [n_dest] zeroed, self-resetting
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
    // fused exchange (decode): wait for this request's SCR_Q (flag of sender b / wait_group),
    // fold the splits in the last CTA of a row, push the packed (O', stats) record to the
    // inquirer's receive slot and raise its flag once all of its rows are in
    const uint32_t* wait_flags;
    int64_t wait_group;
    const uint32_t* epoch;
    uint32_t* fold_counters;   // [n_batch * q_heads * q_rows] zeroed, self-resetting
    float* rec_peer[kMaxPeers];
    uint32_t* rec_flag[kMaxPeers];
    int64_t rec_stride;        // floats per request record (q_heads * q_rows * (d + 2))
    uint32_t* dest_counters;   // [n_dest] zeroed, self-resetting
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
    // fused exchange: wait until wait_flags[0..n_wait) >= *epoch; the last CTA bumps *epoch
    const uint32_t* wait_flags;
    int n_wait;
    uint32_t* epoch;
    uint32_t* done_counter;
};

}  // namespace sda

#include <cuda_runtime.h>
namespace sda {
cudaError_t launch_k1(const K1Params& p, int d, int xdt, int odt, int64_t n_batch, cudaStream_t st);
bool k1_tc_eligible(const K1Params& p, int d, int xdt, int odt);
cudaError_t launch_k1_tc(const K1Params& p, int d, int64_t n_batch, cudaStream_t st);
cudaError_t launch_k2_decode(const K2Params& p, int d, int qdt, int kvdt, cudaStream_t st);
bool k2_prefill_tc_eligible(const K2Params& p, int d, int qdt, int kvdt);
cudaError_t launch_k2_prefill_tc(const K2Params& p, cudaStream_t st);
bool k2_gqa_tc_eligible(const K2Params& p, int d, int qdt, int kvdt);
cudaError_t launch_k2_gqa_tc(const K2Params& p, cudaStream_t st);
cudaError_t launch_k3(const K3Params& p, int d, int odt, cudaStream_t st);

}  // namespace sda
