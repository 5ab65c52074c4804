/*
 * sdattn_b200.h -- C ABI of the B200-native scrambled distributed attention path.
 *
 * This is the drop-in boundary for the reference's hot path (/root/reference/proj/core).
 * Every entry point names the reference interface it replaces (file:line relative to
 * proj/core/). Conventions, chosen to make the ABI bindable from ctypes / cgo / JNI:
 *   - extern "C", plain pointers and sizes, no C++ or torch types, no exceptions;
 *   - every call returns an sda_status mapping the reference's exception cases;
 *   - device buffers are caller-owned; device calls take an explicit cudaStream_t
 *     (passed as void*) and are stream-ordered with no hidden synchronisation;
 *   - no global mutable state: key material lives in caller buffers.
 *
 * Host key derivation (sda_derive_seed .. sda_span_perm) is pure CPU code and is
 * bit-exact with the reference's SplitMix64 / Fisher-Yates / log-uniform draws.
 *
 * Device layouts (row-major, contiguous):
 *   activations / caches : [batch][heads][rows][d]          (bf16 or f32)
 *   partial outputs O'    : [split][batch][q_heads][rows][d] f32
 *   partial stats         : [split][batch][q_heads][rows][2] f32 = (row_max, exp_sum)
 *                           exactly the reference's ShardStats / SCR_SHARD stats frame
 *                           (attention.hpp:38-41, protocol.cpp:1089-1093).
 *   packed key set        : per (request, domain): [kv_heads][2 = {phi_kq, phi_v}] packed
 *                           scramblers, SDA_SCRAMBLER_BYTES(d) each (see sda_pack_keyset).
 */
#ifndef SDATTN_B200_H
#define SDATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDA_ABI_VERSION 1
#define SDA_MAX_SOURCES 64

typedef enum {
    SDA_OK = 0,
    SDA_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument: shapes / ranges (scrambler.cpp:128-130, attention.cpp:32-37) */
    SDA_ERR_NOT_POW2 = 2,         /* build_scrambler: d must be a power of two (scrambler.cpp:27) */
    SDA_ERR_EMPTY_SHARDS = 3,     /* merge_shards: empty shard list (attention.cpp:90) */
    SDA_ERR_MASKED_ROW = 4,       /* merge_shards / attention: row masked in every shard (attention.cpp:99,109-110) */
    SDA_ERR_UNSUPPORTED = 5,      /* valid for the reference but not compiled for the device (e.g. d not in {32,64,128,256}) */
    SDA_ERR_CUDA = 6,             /* a CUDA runtime error (launch / config) */
    SDA_ERR_NO_DEVICE = 7,        /* no sm_100 device visible */
    SDA_ERR_ROLE_VIOLATION = 8,   /* protocol.cpp:215-216: compute node asked for its own domain's keys */
    SDA_ERR_FRAME = 9,            /* FrameError: bad magic / truncated / inconsistent length / CRC mismatch (frame.cpp:138-164) */
    SDA_ERR_TIMEOUT = 10          /* a peer-memory wait gave up (sda_spin_error): a peer rank is gone or far behind */
} sda_status;

/* SDA_F64: the FP64 mode (reference arithmetic and operation order on the device, f64 key image,
 * f64 partials / stats in the float* output slots; SIMT, not a throughput path) of sda_scramble,
 * sda_partial_attention(_causal) and sda_unscramble_merge, and the quantised-wire / frame entry points. */
typedef enum { SDA_BF16 = 0, SDA_F32 = 1, SDA_F64 = 2 } sda_dtype;

/* Which transform of phi a scramble applies (scrambler.cpp:75-85). */
typedef enum {
    SDA_PHI_FORWARD = 0, /* x * phi          : Q (phi_kq) and V (phi_v) */
    SDA_PHI_INV_T = 1,   /* x * phi^{-T}     : K (phi_kq)               */
    SDA_PHI_INV = 2      /* x * phi^{-1}     : O' (phi_v), used by sda_unscramble_merge */
} sda_phi_variant;

typedef enum { SDA_KEYS_KQ = 0, SDA_KEYS_V = 1 } sda_key_which;

typedef enum { SDA_MODE_S1_AND_S2 = 0, SDA_MODE_S1_ONLY = 1 } sda_scrambler_mode; /* scrambler.hpp:33-36 */

/* ------------------------------------------------------------------------------------------
 * Host key derivation -- bit-exact restatement of the protocol key contract.
 * ------------------------------------------------------------------------------------------ */

/* rng.cpp:35-39 derive_seed(base, {tags...}) */
uint64_t sda_derive_seed(uint64_t base, const uint64_t* tags, size_t n_tags);
/* protocol.cpp:143-145 RequestSpec::shared_seed() = derive_seed(master, {request_id, 0x7365656B}) */
uint64_t sda_shared_seed(uint64_t master_seed, uint64_t request_id);
/* permutation.cpp:29-37 random_permutation(n, RngStream(seed)) -> forward[n] */
sda_status sda_random_permutation(size_t n, uint64_t seed, uint32_t* forward);

/* KeySetSpec (scrambler.hpp:77-88) minus l_q/l_k: token permutations are drawn per span. */
typedef struct {
    uint64_t request_id;
    uint32_t layer;
    uint32_t domain;
    uint32_t n_heads;  /* scrambler heads (= kv heads; GQA extension of scrambler.cpp:113-118) */
    uint32_t head_dim; /* power of two */
    double mag_lo;     /* default 0.125 (protocol.hpp:20-27) */
    double mag_hi;     /* default 8.0 */
    int32_t mode;      /* sda_scrambler_mode */
} sda_keyspec;

/* Host key set, f64 factors and u32 permutations exactly as the reference draws them.
 * All arrays [n_heads][head_dim], caller-owned. */
typedef struct {
    double* kq_s1; uint32_t* kq_p1; uint32_t* kq_p2; double* kq_s2;
    double* v_s1;  uint32_t* v_p1;  uint32_t* v_p2;  double* v_s2;
    uint64_t token_perm_seed;
} sda_host_keyset;

/* scrambler.cpp:105-124 negotiate_keyset (feature scramblers + token_perm_seed). */
sda_status sda_negotiate_keyset(uint64_t shared_seed, const sda_keyspec* spec, sda_host_keyset* out);
/* scrambler.cpp:99-103 ScramblerKeySet::span_perm(tag, first_pos, len): tag 0 = Q, 1 = KV. */
sda_status sda_span_perm(uint64_t token_perm_seed, uint64_t tag, uint64_t first_pos, size_t len,
                         uint32_t* forward);
/* inverse permutation: inv[forward[i]] = i (permutation.cpp:15-20) */
sda_status sda_invert_permutation(const uint32_t* forward, size_t n, uint32_t* inverse);

/* Bytes of one packed device scrambler / one head (phi_kq + phi_v) / one key set. */
#define SDA_SCRAMBLER_BYTES(d) ((size_t)34 * (size_t)(d))
#define SDA_KEYSET_HEAD_BYTES(d) ((size_t)68 * (size_t)(d))
size_t sda_keyset_bytes(uint32_t n_heads, uint32_t head_dim);
/* FP64 mode key image (the f64 entry points: x / q / kv / out dtype SDA_F64): raw f64 s1, s2 and
 * the u16 permutations + inverses, so the device repeats the reference's f64 operations exactly. */
#define SDA_SCRAMBLER_BYTES_F64(d) ((size_t)24 * (size_t)(d))
#define SDA_KEYSET_HEAD_BYTES_F64(d) ((size_t)48 * (size_t)(d))
size_t sda_keyset_bytes_f64(uint32_t n_heads, uint32_t head_dim);
sda_status sda_pack_keyset_f64(const sda_host_keyset* ks, uint32_t n_heads, uint32_t head_dim, void* out);
/* Packs a host key set into the device image (f32 factor tables with the 1/sqrt(d) of the
 * normalised FWHT folded in, u16 permutations and their inverses, and the bank-conflict-free
 * order in which K3's warp forms gather through P2 and P1). `out` is host memory of
 * sda_keyset_bytes(); the caller uploads it (cudaMemcpyAsync) next to its other key sets. */
sda_status sda_pack_keyset(const sda_host_keyset* ks, uint32_t n_heads, uint32_t head_dim, void* out);

/* ------------------------------------------------------------------------------------------
 * K1  scramble + token permutation, fused into the cache / wire write.
 *   replaces apply_phi / apply_phi_inv_t + permute_rows_gather (scrambler.cpp:126-136;
 *   protocol.cpp:889-891 for Q, protocol.cpp:998-1001 for the KV write)
 *
 *   out[b][h][out_row_offset + i][:] = x[b][h][perm_b[i]][:] * phi_{b, h / (n_heads/key_heads)}
 *
 *   x    : [n_batch][n_heads][rows][d]              x_dtype
 *   out  : [n_batch][n_heads][out_rows_cap][d]      out_dtype (rounded once, RNE)
 *   keys : device; request b's key set at keys + b * keys_batch_stride (bytes)
 *   perm : device u32; request b's span permutation at perm + b * perm_batch_stride,
 *          NULL = identity (e.g. L_q = 1)
 *   x_batch_mod : 0, or > 0 to read x[b % x_batch_mod] -- one query batch scrambled for several
 *          destination domains (key sets stacked per domain) in a single launch
 * ------------------------------------------------------------------------------------------ */
sda_status sda_scramble(void* stream, int32_t variant, int32_t which_keys,
                        const void* x, int32_t x_dtype, int64_t n_batch, int32_t n_heads,
                        int64_t rows, int32_t head_dim,
                        const void* keys, int64_t keys_batch_stride, int32_t key_heads,
                        const uint32_t* perm, int64_t perm_batch_stride,
                        void* out, int32_t out_dtype, int64_t out_rows_cap, int64_t out_row_offset,
                        int64_t x_batch_mod);

/* K1 with the quantised wire in its epilogue (wire_round, model.cpp:338-341; gen_quant_bits
 * frames, protocol.hpp:25-26): the same scramble + gather as sda_scramble, then every
 * (request, head) tensor of out (rows x d) holds dequantize(quantize_affine(tensor, quant_bits)) of
 * its f32 scrambled values (quant.cpp:26-67: per-tensor min / max, 2..8-bit codes). Two launches of
 * the SIMT K1: a min / max pass and the pass that quantises before its one store (no separate
 * read-modify-write of out). scratch: 2 * n_batch * n_heads u64 device words; err: optional
 * device i32, SDA_ERR_INVALID_ARGUMENT on a non-finite scrambled value (the reference throws). */
sda_status sda_scramble_quant(void* stream, int32_t variant, int32_t which_keys,
                              const void* x, int32_t x_dtype, int64_t n_batch, int32_t n_heads,
                              int64_t rows, int32_t head_dim,
                              const void* keys, int64_t keys_batch_stride, int32_t key_heads,
                              const uint32_t* perm, int64_t perm_batch_stride,
                              void* out, int32_t out_dtype, int64_t out_rows_cap, int64_t out_row_offset,
                              int64_t x_batch_mod, int32_t quant_bits, uint64_t* scratch, int32_t* err);

/* The QKV projection with K1 fused into it (one tcgen05 kernel: projection GEMM -> TMEM -> the
 * scramble as a second GEMM in its epilogue -> bf16 TMA store): replaces project_qkv
 * (model.cpp:124-133) followed by enc_qkv's apply_phi / apply_phi_inv_t + permute_rows_gather
 * (scrambler.cpp:126-136), so no unscrambled Q / K / V reaches HBM.
 *   out[b][h][out_row_offset + r][:] = bf16( (x[b][perm_b[r]][:] . W[h*d .. h*d+d-1][:]^T) phi_{b, h / G} )
 *   x   : bf16 [n_batch][x_rows][d_model]  (the layer input after the norm, model.cpp:124)
 *   w   : bf16 [n_heads * head_dim][d_model], the projection weight as an nn.Linear stores it
 *   out : bf16 [n_batch][n_heads][out_rows_cap][head_dim]; perm as sda_scramble (NULL = identity)
 * head_dim 64 or 128, d_model a multiple of 64; f32 accumulation, one RNE rounding at the store. */
sda_status sda_project_scramble(void* stream, const void* x, int64_t n_batch, int64_t x_rows, int32_t d_model,
                                const void* w, int32_t n_heads, int32_t head_dim, const void* keys,
                                int64_t keys_batch_stride, int32_t key_heads, int32_t variant, int32_t which_keys,
                                const uint32_t* perm, int64_t perm_batch_stride, int64_t rows, void* out,
                                int64_t out_rows_cap, int64_t out_row_offset);

/* Several K1 jobs in one launch (up to SDA_MAX_SCRAMBLE_JOBS; e.g. a prefill step's span K -> K
 * cache, span V -> V cache and Q -> Q'): each job has exactly the meaning of one sda_scramble call
 * with the same fields. When every job takes the tensor-core form (bf16 in/out, head_dim 64 or
 * 128, >= 128 rows) they share one persistent grid, so small spans do not each pay a pipeline
 * fill and a partial last wave; otherwise the jobs run one sda_scramble after another. */
#define SDA_MAX_SCRAMBLE_JOBS 16
typedef struct {
    int32_t variant, which_keys;
    const void* x;
    int32_t x_dtype;
    int64_t n_batch;
    int32_t n_heads;
    int64_t rows;
    const void* keys;
    int64_t keys_batch_stride;
    int32_t key_heads;
    const uint32_t* perm;
    int64_t perm_batch_stride;
    void* out;
    int32_t out_dtype;
    int64_t out_rows_cap, out_row_offset, x_batch_mod;
} sda_scramble_job;
sda_status sda_scramble_batch(void* stream, int32_t head_dim, const sda_scramble_job* jobs, int32_t n_jobs);
/* The same with jobs whose `out` lies in a peer's memory (a receive slot mapped with sda_ipc_*):
 * when all of job j's rows are stored, the CTA completing it raises *peer_flag[j] = *epoch
 * (system-scope release; peer_flag[j] = NULL for a local job). All jobs must take the
 * tensor-core form (else SDA_ERR_UNSUPPORTED). counters: 16 zeroed u32 (self-resetting). This is
 * the prefill SCR_Q send folded into K1 (the span's Q' for every domain written straight into
 * the domains' receive slots, no copy kernel). */
sda_status sda_scramble_batch_remote(void* stream, int32_t head_dim, const sda_scramble_job* jobs, int32_t n_jobs,
                                     uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* counters);

/* ------------------------------------------------------------------------------------------
 * K2  keyless delegated partial attention over the scrambled KV shard.
 *   replaces shard_attention(q', K', V', none) as run by try_serve_q (attention.cpp:42-78;
 *   protocol.cpp:1072-1095). The shard is split along keys into n_splits ranges; every
 *   split emits a locally normalised O' and its (row_max, exp_sum); sda_unscramble_merge
 *   folds splits and nodes in one pass (merge_shards is associative).
 *
 *   q      : [n_batch][q_heads][q_rows][d]  (bf16 or f32; already scrambled)
 *   k, v   : [n_batch][kv_heads][kv_cap][d] (same dtype for k and v)
 *   kv_len : device i32[n_batch] valid rows per request, NULL = kv_cap for all
 *   out_o     : f32 [n_splits][n_batch][q_heads][q_rows][d]
 *   out_stats : f32 [n_splits][n_batch][q_heads][q_rows][2]
 *   q_heads must be a multiple of kv_heads (GQA: q head h reads kv head h / (q_heads/kv_heads)).
 *   Split s covers keys [s*T, min(len, (s+1)*T)) with T = 128 * ceil(ceil(len/128) / n_splits).
 *   The logit scale is 1/sqrt(d) (attention.cpp:45). Rows with no key in a split get
 *   row_max = -inf, exp_sum = 0, O' = 0 (attention.cpp:66-67).
 * ------------------------------------------------------------------------------------------ */
sda_status sda_partial_attention(void* stream, const void* q, int32_t q_dtype,
                                 const void* k, const void* v, int32_t kv_dtype, int64_t kv_cap,
                                 const int32_t* kv_len, int64_t n_batch, int32_t q_heads,
                                 int32_t kv_heads, int64_t q_rows, int32_t head_dim, int32_t n_splits,
                                 float* out_o, float* out_stats);
/* Same, with a workspace for the stream-K form of the tensor-core prefill kernel (n_splits == 1,
 * bf16, d 128, >= 64 query rows): persistent CTAs, one per SM, walk ranges of the key tiles and the
 * pieces of a (request, head, 256-row) unit are merged in the kernel -- full waves without extra
 * partials for K3. workspace: sda_prefill_workspace_bytes() bytes; its first
 * 4 * n_batch * q_heads * ceil(q_rows / 256) bytes are per-unit tickets that must be zero before a
 * launch -- every launch leaves them zero, so a buffer needs zeroing only when it is new or was last
 * used for a larger shape's scratch; the rest is scratch. One workspace serves one launch at a time
 * (e.g. one per stream). workspace == NULL or too small: the split grid, as sda_partial_attention. */
sda_status sda_partial_attention_ws(void* stream, const void* q, int32_t q_dtype,
                                    const void* k, const void* v, int32_t kv_dtype, int64_t kv_cap,
                                    const int32_t* kv_len, int64_t n_batch, int32_t q_heads,
                                    int32_t kv_heads, int64_t q_rows, int32_t head_dim, int32_t n_splits,
                                    float* out_o, float* out_stats, void* workspace, size_t workspace_bytes);
/* Workspace bytes sda_partial_attention_ws needs for this shape; 0 when it does not run stream-K. */
size_t sda_prefill_workspace_bytes(int64_t n_batch, int32_t q_heads, int32_t kv_heads, int64_t q_rows,
                                   int64_t kv_cap, int32_t head_dim, int32_t q_dtype, int32_t kv_dtype);
/* The inquirer's own span is attended in plaintext with a causal mask (protocol.cpp:944-947,
 * AttentionMask::causal(offset), attention.hpp:25-27): key j is visible to query row i iff
 * j <= i + causal_offset. Same layouts and outputs as sda_partial_attention (SIMT kernel). */
sda_status sda_partial_attention_causal(void* stream, const void* q, int32_t q_dtype,
                                        const void* k, const void* v, int32_t kv_dtype, int64_t kv_cap,
                                        const int32_t* kv_len, int64_t n_batch, int32_t q_heads,
                                        int32_t kv_heads, int64_t q_rows, int32_t head_dim, int32_t n_splits,
                                        int64_t causal_offset, float* out_o, float* out_stats);
/* Split count sized for a full-GPU launch of sda_partial_attention (MHA shapes). */
int32_t sda_default_splits(int64_t n_batch, int32_t q_heads, int64_t q_rows, int64_t kv_cap);
/* Same, aware of GQA (q_heads > kv_heads) and of which kernel the shape dispatches to. */
int32_t sda_default_splits_gqa(int64_t n_batch, int32_t q_heads, int32_t kv_heads, int64_t q_rows,
                               int64_t kv_cap, int32_t head_dim);

/* ------------------------------------------------------------------------------------------
 * K3  cross-node LSE-weighted merge + inverse token permutation + unscramble.
 *   replaces dec_output (scrambler.cpp:138-149) for every remote shard followed by
 *   merge_shards (attention.cpp:89-123), as span_finish_layer does (protocol.cpp:926-948).
 *
 *   Source s contributes rows o_s[b][h][pq_inv_s[b][r]] (its rows are in its domain's P_Q
 *   order) with stats stats_s. Sources with the same `keys` pointer form one group: their
 *   weighted sum is unscrambled once with that group's phi_v^{-1} (linearity). keys == NULL
 *   marks a plaintext source (e.g. the inquirer's local shard). A single source is returned
 *   unweighted, as merge_shards returns one shard verbatim (attention.cpp:97-101).
 *
 *   out       : [n_batch][q_heads][q_rows][d] out_dtype
 *   out_stats : optional f32 [n_batch][q_heads][q_rows][2] merged (row_max, exp_sum), may be NULL
 *   err_flag  : optional device i32; set to SDA_ERR_MASKED_ROW when a row has exp_sum == 0 in
 *               every source (that row is written as NaN). May be NULL.
 *   out_batch_stride : elements between requests in out and out_stats (0 = dense); a packed
 *               per-request record [q_heads*q_rows*d | q_heads*q_rows*2] is what one NCCL
 *               all-to-all carries back to the inquirer (O' and stats together).
 *   alignment (d >= 32, f32 / bf16 out): every O' and output row is moved as one d/32-element
 *               vector per lane, so source and output pointers and batch strides must keep rows
 *               aligned to that vector (min(16, 4 d/32) bytes for O', min(16, d/32 sizeof(out))
 *               for out) and stats pairs to 8 bytes; otherwise SDA_ERR_INVALID_ARGUMENT. A packed
 *               record qualifies whenever q_heads * q_rows is even.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
    const float* o;          /* [n_batch][q_heads][q_rows][d] */
    const float* stats;      /* [n_batch][q_heads][q_rows][2] */
    const void* keys;        /* device key set of the domain (phi_v used), NULL = plaintext */
    const uint32_t* pq_inv;  /* device u32 inverse span perm per request, NULL = identity */
    int64_t batch_stride;    /* elements between requests in o and stats (0 = dense as above);
                                lets O' and stats share one packed per-request record */
} sda_merge_source;

sda_status sda_unscramble_merge(void* stream, const sda_merge_source* sources, int32_t n_sources,
                                int64_t keys_batch_stride, int32_t key_heads, int64_t pq_batch_stride,
                                int64_t n_batch, int32_t q_heads, int64_t q_rows, int32_t head_dim,
                                void* out, int32_t out_dtype, float* out_stats, int32_t* err_flag,
                                int64_t out_batch_stride);

/* K3 with the quantised O' wire on its input path (SCR_SHARD frames in quantN, protocol.hpp:25-26;
 * wire_round of O', model.cpp:392): the same merge as sda_unscramble_merge, except that every key
 * group's O' -- the domain's normalised partial, still scrambled -- is replaced by
 * dequantize(quantize_affine(O', quant_bits)) per (request, head) tensor (q_rows x d) before its
 * unscramble; the stats stay f32 (wire_round_stat). One query row: a single launch (the warp holds
 * the whole tensor); more rows: a min / max pass first, scratch = 2 * groups * n_batch * q_heads
 * u64 device words (groups = runs of sources sharing a key set). head_dim >= 32, out bf16 / f32. */
sda_status sda_unscramble_merge_quant(void* stream, const sda_merge_source* sources, int32_t n_sources,
                                      int64_t keys_batch_stride, int32_t key_heads, int64_t pq_batch_stride,
                                      int64_t n_batch, int32_t q_heads, int64_t q_rows, int32_t head_dim,
                                      void* out, int32_t out_dtype, float* out_stats, int32_t* err_flag,
                                      int64_t out_batch_stride, int32_t quant_bits, uint64_t* scratch);

/* ------------------------------------------------------------------------------------------
 * Peer-memory exchange (replaces Simulator::send of SCR_Q / SCR_SHARD, protocol.cpp:892-896,
 * :1097-1102, inside one NVSwitch box). Receive buffers are mapped into every peer with CUDA
 * IPC; a push copies each peer's payload over NVLink and raises that peer's per-sender flag
 * (system-scope release) with the step epoch; a wait spins (acquire) until all of its flags
 * reached the epoch. All stream-ordered and graph-capturable. No wait hangs or traps: one that sees
 * nothing within the spin budget (sda_set_spin_timeout_ns, default 30 s) returns and records
 * SDA_ERR_TIMEOUT, which sda_spin_error reports; the exchange must then be torn down.
 * ------------------------------------------------------------------------------------------ */
/* handle_out: 64 bytes (cudaIpcMemHandle_t of the allocation containing dev_ptr) + offset in it */
sda_status sda_ipc_get_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out);
sda_status sda_ipc_open_handle(const void* handle, uint64_t offset, void** dev_ptr_out);
sda_status sda_ipc_close_handle(void* dev_ptr, uint64_t offset);
/* *epoch += 1 (one per step, before the pushes / waits of that step) */
sda_status sda_exchange_epoch(void* stream, uint32_t* epoch);
/* for p < n_peers: copy bytes (multiple of 16) src[p] -> dst[p], then *peer_flags[p] = *epoch.
 * counters: n_peers zero-initialised device u32 (self-resetting). */
sda_status sda_exchange_push(void* stream, int32_t n_peers, const void* const* src, void* const* dst,
                             uint32_t* const* peer_flags, uint64_t bytes, const uint32_t* epoch,
                             uint32_t* counters);
/* wait until flags[i] >= *epoch for i < n (wrap-around safe) */
sda_status sda_exchange_wait(void* stream, const uint32_t* flags, int32_t n, const uint32_t* epoch);
/* Spin budget (ns) of every peer-memory wait on the current device (synchronous; default 30 s). */
sda_status sda_set_spin_timeout_ns(uint64_t ns);
/* *out = SDA_ERR_TIMEOUT if a wait on the current device gave up since the last clear, else SDA_OK
 * (synchronous: call between steps, e.g. after a stream synchronize); clear != 0 resets it. */
sda_status sda_spin_error(int32_t* out, int32_t clear);

/* LL exchange for single-row decode (L_q = 1, head_dim >= 64): the three kernels of a step carry
 * the exchange themselves over peer memory (buffers mapped with sda_ipc_*), so a step is 3
 * launches with no copy kernel, fence or flag: every 4-byte data word travels next to the 4-byte
 * step epoch ("LL" format, 16-byte stores of two (word, epoch) pairs) and readers spin until their
 * words carry the current *epoch (spin budget and error reporting as above). *epoch starts at 1 with
 * all receive buffers zeroed; sda_ll_unscramble_merge bumps it when it finishes.
 *
 * Receive buffers on every rank (W = ranks, B_p = requests per inquirer, H = q heads, d):
 *   Q' slots     [W senders][B_p][H][d]      LL: bf16 wire 4 B per element, f32 wire 8 B per element
 *   record slots [W senders][S splits][B_p][H][d + 2]   LL f32: 8 B per float ([d O' | row_max, exp_sum])
 *
 * sda_ll_scramble_q: K1 (phi_KQ forward) of q [B_p][H][1][d] with the key set of request
 *   dest * B_p + b (keys stacked destination-major) into ll_q[dest] = destination's Q' slot for
 *   this sender. */
sda_status sda_ll_scramble_q(void* stream, const void* q, int32_t q_dtype, int32_t n_dest, int64_t b_per,
                             int32_t n_heads, int32_t head_dim, const void* keys, int64_t keys_batch_stride,
                             int32_t key_heads, void* const* ll_q, int32_t wire_dtype, const uint32_t* epoch);
/* sda_ll_partial_attention: K2 over this rank's Q' slots (ll_q = [W][B_p][H][d] LL) and its KV
 *   shard (requests sender-major, kv_len / k / v as sda_partial_attention); split s of request
 *   (sender, i) goes to ll_rec[sender] = the sender's record slot for this domain.
 *   gqa_work: optional device buffer of W * B_p * H * d bf16; with it, GQA shards (bf16, d 128,
 *   2 <= H / kv_heads <= 32) run the tensor-core GQA kernel (Q' unpacked from LL first). */
sda_status sda_ll_partial_attention(void* stream, const void* ll_q, int32_t wire_dtype, const void* k, const void* v,
                                    int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int32_t n_dest,
                                    int64_t b_per, int32_t q_heads, int32_t kv_heads, int32_t head_dim,
                                    int32_t n_splits, void* const* ll_rec, const uint32_t* epoch, void* gqa_work);
/* Remote records for prefill spans (q_rows >= 64, tensor-core form, one split): K2 over
 *   q [n_dest * b_per][q_heads][q_rows][d] (requests sender-major) writing request (dest, i)'s
 *   packed record [q_heads * q_rows * d O' | q_heads * q_rows * 2 stats] straight into
 *   rec_peer[dest] + i * rec_stride floats (the inquirer's receive slot, peer memory); the CTA
 *   completing a destination raises *peer_flag[dest] = *epoch (system-scope release), which the
 *   inquirer's sda_exchange_wait consumes. Replaces K2 + split fold + sda_exchange_push on the
 *   return path. dest_counters: n_dest zeroed u32 (self-resetting). workspace / workspace_bytes:
 *   as sda_partial_attention_ws (stream-K; NULL -> the split grid). */
sda_status sda_partial_attention_remote(void* stream, const void* q, int32_t q_dtype, const void* k, const void* v,
                                        int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int32_t n_dest,
                                        int64_t b_per, int32_t q_heads, int32_t kv_heads, int64_t q_rows,
                                        int32_t head_dim, float* const* rec_peer, int64_t rec_stride,
                                        uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* dest_counters,
                                        void* workspace, size_t workspace_bytes);
/* sda_ll_unscramble_merge: K3 over this rank's record slots (n_domains * n_splits sources, each
 *   domain unscrambled with its phi_V^-1 from keys[(domain * B_p + b)]) into out [B_p][H][1][d];
 *   then *epoch += 1. done_counter: one zeroed u32 (self-resetting). */
sda_status sda_ll_unscramble_merge(void* stream, const void* ll_rec, int32_t n_domains, int32_t n_splits,
                                   const void* keys, int64_t keys_batch_stride, int32_t key_heads, int64_t b_per,
                                   int32_t q_heads, int32_t head_dim, void* out, int32_t out_dtype, uint32_t* epoch,
                                   uint32_t* done_counter);

/* Step tracing: *dst = the GPU's %globaltimer (ns) when this 1-thread kernel runs, in stream
 * order. Not counted by sda_launch_count (instrumentation, not part of a step). */
sda_status sda_trace_timestamp(void* stream, uint64_t* dst);

/* ------------------------------------------------------------------------------------------
 * Quantised wire (quant.cpp:26-67; wire_round model.cpp:338-341; gen_quant_bits
 * protocol.hpp:25-26): per-tensor affine min-max quantisation, 2..8-bit codes packed LSB-first,
 * bit-exact with quantize_affine / dequantize on the same input values. n_tensors contiguous
 * tensors of `count` elements each (x, out: [n_tensors][count]); x / out dtype SDA_F32, SDA_F64
 * or SDA_BF16. scratch: 2 * n_tensors u64 device words. err: optional device i32, set to
 * SDA_ERR_INVALID_ARGUMENT on a non-finite input value (the reference throws).
 * ------------------------------------------------------------------------------------------ */
/* codes of tensor t at codes + t * codes_stride (>= ceil(count * bits / 8) bytes, unused bits 0);
 * scale[t], zero_point[t] as the reference's QTensor (f32) */
sda_status sda_quantize_affine(void* stream, const void* x, int32_t x_dtype, int64_t n_tensors, int64_t count,
                               int32_t bits, uint8_t* codes, int64_t codes_stride, float* scale, float* zero_point,
                               uint64_t* scratch, int32_t* err);
sda_status sda_dequantize(void* stream, const uint8_t* codes, int64_t codes_stride, const float* scale,
                          const float* zero_point, int64_t n_tensors, int64_t count, int32_t bits, void* out,
                          int32_t out_dtype);
/* x <- dequantize(quantize_affine(x, bits)) per tensor, in place (the wire emulation) */
sda_status sda_quant_roundtrip(void* stream, void* x, int32_t dtype, int64_t n_tensors, int64_t count, int32_t bits,
                               uint64_t* scratch, int32_t* err);

/* x <- round_to_format(x, wire_fmt) in place, the float-format wire_round (float_format.cpp:26-58,
 * model.cpp:339-348, protocol.cpp:179): RNE onto the format's grid done in f64, +-inf and overflow
 * clamped to +-max_finite. x: n device values, x_dtype SDA_F32 or SDA_F64; wire_fmt the reference's
 * FloatFormat (0 f64 = no-op, 1 f32, 2 bf16, 3 f16). */
sda_status sda_wire_round(void* stream, void* x, int32_t x_dtype, int64_t n, int32_t wire_fmt);

/* ------------------------------------------------------------------------------------------
 * Wire frames on the device ("FATN", frame.hpp:48-92): encode a device tensor into the
 * reference's bit-exact frame bytes, CRC-32 included, and decode one back.
 *   dtype: the reference's DtypeCode -- 0 f64, 1 f32, 2 bf16, 3 f16, 16+N quantN (N = 2..8).
 *   Tensor frames (make_tensor_frame) carry dims {n_tensors, rows, cols}; any dims (<= 8) work.
 * ------------------------------------------------------------------------------------------ */
#define SDA_FRAME_MAX_DIMS 8
typedef struct {
    uint8_t version;      /* 1 */
    uint8_t msg_type;     /* MsgType: 2 SCR_KV, 3 SCR_Q, 4 SCR_SHARD, ... */
    uint64_t request_id;
    uint16_t layer, head, domain;
    uint8_t dtype;        /* DtypeCode */
    uint32_t n_dims;
    uint32_t dims[SDA_FRAME_MAX_DIMS];
} sda_frame_header;
/* element count (0 without dims), payload bytes (dtype_payload_size, frame.cpp:63-75), whole frame
 * (encoded_size, frame.cpp:134-136), device scratch for sda_frame_encode / _decode / sda_crc32 */
uint64_t sda_frame_elements(const sda_frame_header* h);
uint64_t sda_frame_payload_bytes(const sda_frame_header* h);
uint64_t sda_frame_bytes(const sda_frame_header* h);
uint64_t sda_frame_scratch_bytes(uint64_t frame_bytes);
/* payload_from_values + encode_frame: x (device, x_dtype SDA_F32 / SDA_F64 / SDA_BF16, the
 * frame's elements in order) -> out (device, sda_frame_bytes(h) bytes). err: optional device
 * i32, SDA_ERR_INVALID_ARGUMENT on a non-finite value for a quantN frame. */
sda_status sda_frame_encode(void* stream, const sda_frame_header* h, const void* x, int32_t x_dtype, uint8_t* out,
                            void* scratch, int32_t* err);
/* host: the header fields and length checks of decode_frame (magic, truncation, payload length,
 * frame.cpp:138-158) from the first bytes of a frame (size = the whole frame's length) */
sda_status sda_frame_parse_header(const uint8_t* host_bytes, uint64_t host_len, uint64_t frame_size,
                                  sda_frame_header* out);
/* decode_frame's CRC check + values_from_payload: frame (device, frame_size bytes, header h as
 * parsed) -> out (device, out_dtype). A CRC mismatch sets *err = SDA_ERR_FRAME. */
sda_status sda_frame_decode(void* stream, const uint8_t* frame, uint64_t frame_size, const sda_frame_header* h,
                            void* out, int32_t out_dtype, void* scratch, int32_t* err);
/* CRC-32/IEEE of len device bytes (crc32, frame.cpp:78-83) -> out4 (device, little-endian) */
sda_status sda_crc32(void* stream, const uint8_t* bytes, uint64_t len, void* scratch, uint8_t* out4);

/* ------------------------------------------------------------------------------------------
 * Misc
 * ------------------------------------------------------------------------------------------ */
int32_t sda_abi_version(void);
const char* sda_status_string(int32_t status);
/* Number of kernel launches issued by this library since load (for bench gpu_launches). */
uint64_t sda_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SDATTN_B200_H */
