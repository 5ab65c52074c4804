// capi.cu -- the extern "C" boundary (include/sdattn_b200.h): argument validation that
// mirrors the reference's std::invalid_argument cases, then stream-ordered kernel launches.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace {

std::atomic<uint64_t> g_launches{0};

}  // namespace

namespace sda {
void count_launch() { ++g_launches; }
}  // namespace sda

namespace {

// 4..16: SIMT forms for the reference's own small-model tests; 32..256: every form
bool supported_dim(int d) { return d == 4 || d == 8 || d == 16 || d == 32 || d == 64 || d == 128 || d == 256; }
bool pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
// Debug knobs (tests compare kernel variants): SDA_K1_SIMT=1 / SDA_K2_SIMT=1 force the SIMT
// K1 / K2 kernels; SDA_K2_GROUPED=1 routes small GQA groups to the grouped-row kernel.
bool env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] && v[0] != '0';
}

bool valid_dtype(int t) { return t == SDA_BF16 || t == SDA_F32; }
size_t dtype_size(int t) { return t == SDA_BF16 ? 2 : t == SDA_F32 ? 4 : 8; }
// rows of d elements are moved as vectors of up to 16 bytes: the base pointer must be aligned to
// min(16, one row) (row strides are whole rows, so every row then is)
bool row_aligned(const void* ptr, int d, int dt) {
    const uintptr_t a = std::min<size_t>(16, (size_t)d * dtype_size(dt));
    return reinterpret_cast<uintptr_t>(ptr) % a == 0;
}
// FP64 mode (f64_path.cu): every tensor of the call f64, or none
bool valid_dtype_f64(int t) { return valid_dtype(t) || t == SDA_F64; }
bool f64_pair_ok(int a, int b) { return (a == SDA_F64) == (b == SDA_F64); }

sda_status from_cuda(cudaError_t e) {
    if (e == cudaSuccess) return SDA_OK;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SDA_ERR_NO_DEVICE;
    return SDA_ERR_CUDA;
}

}  // namespace

extern "C" {

static sda_status unscramble_merge_impl(void* stream, const sda_merge_source* sources, int32_t n_sources,
                                        int64_t keys_batch_stride, int32_t key_heads, int64_t pq_batch_stride,
                                        int64_t n_batch, int32_t q_heads, int64_t q_rows, int32_t head_dim, void* out,
                                        int32_t out_dtype, float* out_stats, int32_t* err_flag,
                                        int64_t out_batch_stride, int quant_bits, int n_groups,
                                        unsigned long long* qscratch);

int32_t sda_abi_version(void) { return SDA_ABI_VERSION; }

uint64_t sda_launch_count(void) { return g_launches.load(); }

const char* sda_status_string(int32_t s) {
    switch (s) {
        case SDA_OK: return "ok";
        case SDA_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SDA_ERR_NOT_POW2: return "head dim must be a power of two";
        case SDA_ERR_EMPTY_SHARDS: return "merge: empty shard list";
        case SDA_ERR_MASKED_ROW: return "merge: row masked in every shard";
        case SDA_ERR_UNSUPPORTED: return "unsupported on device (head dim not in {4,8,16,32,64,128,256}, or a form that needs d >= 64)";
        case SDA_ERR_CUDA: return "CUDA error";
        case SDA_ERR_NO_DEVICE: return "no CUDA device";
        case SDA_ERR_ROLE_VIOLATION: return "role violation";
        case SDA_ERR_FRAME: return "frame error (magic / length / dtype / CRC)";
        case SDA_ERR_TIMEOUT: return "peer-memory wait timed out (a peer rank is gone or far behind)";
        default: return "unknown status";
    }
}

sda_status sda_scramble(void* stream, int32_t variant, int32_t which_keys, const void* x, int32_t x_dtype,
                        int64_t n_batch, int32_t n_heads, int64_t rows, int32_t head_dim, const void* keys,
                        int64_t keys_batch_stride, int32_t key_heads, const uint32_t* perm,
                        int64_t perm_batch_stride, void* out, int32_t out_dtype, int64_t out_rows_cap,
                        int64_t out_row_offset, int64_t x_batch_mod) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    if (variant != SDA_PHI_FORWARD && variant != SDA_PHI_INV_T) return SDA_ERR_INVALID_ARGUMENT;
    if (which_keys != SDA_KEYS_KQ && which_keys != SDA_KEYS_V) return SDA_ERR_INVALID_ARGUMENT;
    if (!x || !out || !keys || !valid_dtype_f64(x_dtype) || !valid_dtype_f64(out_dtype) || !f64_pair_ok(x_dtype, out_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if (!row_aligned(x, head_dim, x_dtype) || !row_aligned(out, head_dim, out_dtype)) return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch < 0 || n_heads <= 0 || key_heads <= 0 || n_heads % key_heads != 0 || rows < 0)
        return SDA_ERR_INVALID_ARGUMENT;
    if (out_row_offset < 0 || out_row_offset + rows > out_rows_cap || x_batch_mod < 0) return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch > 65535 || n_heads > 65535) return SDA_ERR_UNSUPPORTED;
    if (rows == 0 || n_batch == 0) return SDA_OK;
    sda::K1Params p{x, out, keys, perm, keys_batch_stride, perm_batch_stride, rows, out_rows_cap, out_row_offset,
                    n_heads, key_heads, which_keys, variant == SDA_PHI_INV_T ? 1 : 0, x_batch_mod};
    ++g_launches;
    if (x_dtype == SDA_F64)
        return from_cuda(sda::launch_f64_path(1, &p, head_dim, n_batch, static_cast<cudaStream_t>(stream)));
    if (sda::k1_tc_eligible(p, head_dim, x_dtype, out_dtype) && !env_flag("SDA_K1_SIMT"))
        return from_cuda(sda::launch_k1_tc(p, head_dim, n_batch, static_cast<cudaStream_t>(stream)));
    return from_cuda(sda::launch_k1(p, head_dim, x_dtype, out_dtype, n_batch, static_cast<cudaStream_t>(stream)));
}

sda_status sda_scramble_quant(void* stream, int32_t variant, int32_t which_keys, const void* x, int32_t x_dtype,
                              int64_t n_batch, int32_t n_heads, int64_t rows, int32_t head_dim, const void* keys,
                              int64_t keys_batch_stride, int32_t key_heads, const uint32_t* perm,
                              int64_t perm_batch_stride, void* out, int32_t out_dtype, int64_t out_rows_cap,
                              int64_t out_row_offset, int64_t x_batch_mod, int32_t quant_bits, uint64_t* scratch,
                              int32_t* err) {
    if (quant_bits < 2 || quant_bits > 8) return SDA_ERR_INVALID_ARGUMENT;   // quant.cpp:27
    if (!scratch) return SDA_ERR_INVALID_ARGUMENT;
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    if (variant != SDA_PHI_FORWARD && variant != SDA_PHI_INV_T) return SDA_ERR_INVALID_ARGUMENT;
    if (which_keys != SDA_KEYS_KQ && which_keys != SDA_KEYS_V) return SDA_ERR_INVALID_ARGUMENT;
    if (!x || !out || !keys || !valid_dtype(x_dtype) || !valid_dtype(out_dtype)) return SDA_ERR_INVALID_ARGUMENT;
    if (!row_aligned(x, head_dim, x_dtype) || !row_aligned(out, head_dim, out_dtype)) return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch < 0 || n_heads <= 0 || key_heads <= 0 || n_heads % key_heads != 0 || rows < 0)
        return SDA_ERR_INVALID_ARGUMENT;
    if (out_row_offset < 0 || out_row_offset + rows > out_rows_cap || x_batch_mod < 0) return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch > 65535 || n_heads > 65535) return SDA_ERR_UNSUPPORTED;
    if (rows == 0 || n_batch == 0) return SDA_OK;
    sda::K1Params p{x, out, keys, perm, keys_batch_stride, perm_batch_stride, rows, out_rows_cap, out_row_offset,
                    n_heads, key_heads, which_keys, variant == SDA_PHI_INV_T ? 1 : 0, x_batch_mod};
    p.quant_bits = quant_bits;
    p.qscratch = reinterpret_cast<unsigned long long*>(scratch);
    p.qerr = err;
    g_launches += 2;
    return from_cuda(sda::launch_k1(p, head_dim, x_dtype, out_dtype, n_batch, static_cast<cudaStream_t>(stream)));
}

sda_status sda_project_scramble(void* stream, const void* x, int64_t n_batch, int64_t x_rows, int32_t d_model,
                                const void* w, int32_t n_heads, int32_t head_dim, const void* keys,
                                int64_t keys_batch_stride, int32_t key_heads, int32_t variant, int32_t which_keys,
                                const uint32_t* perm, int64_t perm_batch_stride, int64_t rows, void* out,
                                int64_t out_rows_cap, int64_t out_row_offset) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (head_dim != 64 && head_dim != 128) return SDA_ERR_UNSUPPORTED;
    if (d_model <= 0 || d_model % 64 != 0) return SDA_ERR_UNSUPPORTED;
    if (variant != SDA_PHI_FORWARD && variant != SDA_PHI_INV_T) return SDA_ERR_INVALID_ARGUMENT;
    if (which_keys != SDA_KEYS_KQ && which_keys != SDA_KEYS_V) return SDA_ERR_INVALID_ARGUMENT;
    if (!x || !w || !keys || !out || n_batch < 0 || x_rows < 0 || rows < 0 || n_heads <= 0 || key_heads <= 0 ||
        n_heads % key_heads != 0)
        return SDA_ERR_INVALID_ARGUMENT;
    if (!perm && rows > x_rows) return SDA_ERR_INVALID_ARGUMENT;
    if (out_row_offset < 0 || out_row_offset + rows > out_rows_cap) return SDA_ERR_INVALID_ARGUMENT;
    if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(w) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
        return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch > 65535 || n_heads > 65535) return SDA_ERR_UNSUPPORTED;
    if (rows == 0 || n_batch == 0) return SDA_OK;
    ++g_launches;
    return from_cuda(sda::launch_project_scramble(x, n_batch, x_rows, d_model, w, n_heads, head_dim, keys,
                                                  keys_batch_stride, key_heads, variant, which_keys, perm,
                                                  perm_batch_stride, rows, out, out_rows_cap, out_row_offset,
                                                  static_cast<cudaStream_t>(stream)));
}

static sda_status scramble_batch_impl(void* stream, int32_t head_dim, const sda_scramble_job* jobs, int32_t n_jobs,
                                      uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* counters) {
    if (!jobs || n_jobs < 0 || n_jobs > SDA_MAX_SCRAMBLE_JOBS) return SDA_ERR_INVALID_ARGUMENT;
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    const bool remote = peer_flag != nullptr;
    if (remote && (!epoch || !counters)) return SDA_ERR_INVALID_ARGUMENT;
    sda::K1Params ps[SDA_MAX_SCRAMBLE_JOBS];
    int64_t nb[SDA_MAX_SCRAMBLE_JOBS];
    uint32_t* flags[SDA_MAX_SCRAMBLE_JOBS];
    int n_live = 0;
    bool all_tc = !env_flag("SDA_K1_SIMT");
    for (int i = 0; i < n_jobs; ++i) {   // same validation as sda_scramble, per job
        const sda_scramble_job& j = jobs[i];
        if (j.variant != SDA_PHI_FORWARD && j.variant != SDA_PHI_INV_T) return SDA_ERR_INVALID_ARGUMENT;
        if (j.which_keys != SDA_KEYS_KQ && j.which_keys != SDA_KEYS_V) return SDA_ERR_INVALID_ARGUMENT;
        if (!j.x || !j.out || !j.keys || !valid_dtype_f64(j.x_dtype) || !valid_dtype_f64(j.out_dtype) ||
            !f64_pair_ok(j.x_dtype, j.out_dtype))
            return SDA_ERR_INVALID_ARGUMENT;
        if (j.n_batch < 0 || j.n_heads <= 0 || j.key_heads <= 0 || j.n_heads % j.key_heads != 0 || j.rows < 0)
            return SDA_ERR_INVALID_ARGUMENT;
        if (j.out_row_offset < 0 || j.out_row_offset + j.rows > j.out_rows_cap || j.x_batch_mod < 0)
            return SDA_ERR_INVALID_ARGUMENT;
        if (j.n_batch > 65535 || j.n_heads > 65535) return SDA_ERR_UNSUPPORTED;
        if (j.rows == 0 || j.n_batch == 0) {
            if (remote && peer_flag[i]) return SDA_ERR_INVALID_ARGUMENT;   // an empty remote job would never signal
            continue;
        }
        sda::K1Params p{j.x, j.out, j.keys, j.perm, j.keys_batch_stride, j.perm_batch_stride, j.rows, j.out_rows_cap,
                        j.out_row_offset, j.n_heads, j.key_heads, j.which_keys, j.variant == SDA_PHI_INV_T ? 1 : 0,
                        j.x_batch_mod};
        all_tc = all_tc && sda::k1_tc_eligible(p, head_dim, j.x_dtype, j.out_dtype);
        ps[n_live] = p;
        nb[n_live] = j.n_batch;
        flags[n_live] = remote ? peer_flag[i] : nullptr;
        ++n_live;
    }
    if (n_live == 0) return SDA_OK;
    if (all_tc) {
        ++g_launches;
        return from_cuda(sda::launch_k1_tc_multi(ps, nb, n_live, head_dim, static_cast<cudaStream_t>(stream),
                                                 remote ? flags : nullptr, remote ? epoch : nullptr,
                                                 remote ? counters : nullptr));
    }
    if (remote) return SDA_ERR_UNSUPPORTED;
    for (int i = 0; i < n_jobs; ++i) {
        const sda_scramble_job& j = jobs[i];
        const sda_status st = sda_scramble(stream, j.variant, j.which_keys, j.x, j.x_dtype, j.n_batch, j.n_heads, j.rows,
                                           head_dim, j.keys, j.keys_batch_stride, j.key_heads, j.perm,
                                           j.perm_batch_stride, j.out, j.out_dtype, j.out_rows_cap, j.out_row_offset,
                                           j.x_batch_mod);
        if (st != SDA_OK) return st;
    }
    return SDA_OK;
}

sda_status sda_scramble_batch(void* stream, int32_t head_dim, const sda_scramble_job* jobs, int32_t n_jobs) {
    return scramble_batch_impl(stream, head_dim, jobs, n_jobs, nullptr, nullptr, nullptr);
}

sda_status sda_scramble_batch_remote(void* stream, int32_t head_dim, const sda_scramble_job* jobs, int32_t n_jobs,
                                     uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* counters) {
    if (!peer_flag) return SDA_ERR_INVALID_ARGUMENT;
    return scramble_batch_impl(stream, head_dim, jobs, n_jobs, peer_flag, epoch, counters);
}

// ------------------------------------------------------------------------------------------ quant wire
static bool quant_dtype_ok(int t) { return t == SDA_BF16 || t == SDA_F32 || t == SDA_F64; }

sda_status sda_quantize_affine(void* stream, const void* x, int32_t x_dtype, int64_t n_tensors, int64_t count,
                               int32_t bits, uint8_t* codes, int64_t codes_stride, float* scale, float* zero_point,
                               uint64_t* scratch, int32_t* err) {
    if (bits < 2 || bits > 8) return SDA_ERR_INVALID_ARGUMENT;   // quant.cpp:27
    if (n_tensors < 0 || count < 0 || !quant_dtype_ok(x_dtype) || n_tensors > 65535) return SDA_ERR_INVALID_ARGUMENT;
    if (n_tensors == 0) return SDA_OK;
    if (!x || !codes || !scale || !zero_point || !scratch || codes_stride < (count * bits + 7) / 8)
        return SDA_ERR_INVALID_ARGUMENT;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (count == 0) {   // empty tensor: scale 0, zero point 0, no codes (quant.cpp:33)
        cudaError_t e = cudaMemsetAsync(scale, 0, n_tensors * 4, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(zero_point, 0, n_tensors * 4, st);
        return from_cuda(e);
    }
    g_launches += 2;
    return from_cuda(sda::launch_quantize(x, x_dtype, n_tensors, count, bits, codes, codes_stride, scale, zero_point,
                                          reinterpret_cast<unsigned long long*>(scratch), err, st));
}

sda_status sda_dequantize(void* stream, const uint8_t* codes, int64_t codes_stride, const float* scale,
                          const float* zero_point, int64_t n_tensors, int64_t count, int32_t bits, void* out,
                          int32_t out_dtype) {
    if (bits < 2 || bits > 8) return SDA_ERR_INVALID_ARGUMENT;
    if (n_tensors < 0 || count < 0 || !quant_dtype_ok(out_dtype) || n_tensors > 65535) return SDA_ERR_INVALID_ARGUMENT;
    if (n_tensors == 0 || count == 0) return SDA_OK;
    if (!codes || !scale || !zero_point || !out || codes_stride < (count * bits + 7) / 8) return SDA_ERR_INVALID_ARGUMENT;
    ++g_launches;
    return from_cuda(sda::launch_dequantize(codes, codes_stride, scale, zero_point, n_tensors, count, bits, out,
                                            out_dtype, static_cast<cudaStream_t>(stream)));
}

sda_status sda_quant_roundtrip(void* stream, void* x, int32_t dtype, int64_t n_tensors, int64_t count, int32_t bits,
                               uint64_t* scratch, int32_t* err) {
    if (bits < 2 || bits > 8) return SDA_ERR_INVALID_ARGUMENT;
    if (n_tensors < 0 || count < 0 || !quant_dtype_ok(dtype) || n_tensors > 65535) return SDA_ERR_INVALID_ARGUMENT;
    if (n_tensors == 0 || count == 0) return SDA_OK;
    if (!x || !scratch) return SDA_ERR_INVALID_ARGUMENT;
    g_launches += 2;
    return from_cuda(sda::launch_quant_roundtrip(x, dtype, n_tensors, count, bits,
                                                 reinterpret_cast<unsigned long long*>(scratch), err,
                                                 static_cast<cudaStream_t>(stream)));
}

sda_status sda_wire_round(void* stream, void* x, int32_t x_dtype, int64_t n, int32_t wire_fmt) {
    if (n < 0 || (x_dtype != SDA_F32 && x_dtype != SDA_F64) || wire_fmt < 0 || wire_fmt > 3)
        return SDA_ERR_INVALID_ARGUMENT;
    if (n == 0 || wire_fmt == 0) return SDA_OK;
    if (!x) return SDA_ERR_INVALID_ARGUMENT;
    ++g_launches;
    return from_cuda(sda::launch_wire_round(x, x_dtype, n, wire_fmt, static_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------------------------------ frames
static bool frame_dtype_ok(int d) { return (d >= 0 && d <= 3) || (d >= 18 && d <= 24); }

uint64_t sda_frame_elements(const sda_frame_header* h) {
    if (!h || h->n_dims == 0 || h->n_dims > SDA_FRAME_MAX_DIMS) return 0;
    uint64_t n = 1;
    for (uint32_t i = 0; i < h->n_dims; ++i) n *= h->dims[i];
    return n;
}

uint64_t sda_frame_payload_bytes(const sda_frame_header* h) {
    if (!h || !frame_dtype_ok(h->dtype)) return 0;
    const uint64_t n = sda_frame_elements(h);
    switch (h->dtype) {
        case 0: return n * 8;
        case 1: return n * 4;
        case 2:
        case 3: return n * 2;
        default: return (n * (uint64_t)(h->dtype - 16) + 7) / 8 + 8;
    }
}

static uint64_t frame_header_bytes(const sda_frame_header* h) { return 25 + 4ull * h->n_dims; }

uint64_t sda_frame_bytes(const sda_frame_header* h) {
    if (!h || h->n_dims > SDA_FRAME_MAX_DIMS) return 0;
    return frame_header_bytes(h) + sda_frame_payload_bytes(h) + 4;
}

uint64_t sda_frame_scratch_bytes(uint64_t frame_bytes) {
    return ((sda::crc_scratch_words(frame_bytes) * 4 + 255) / 256) * 256 + 256;
}

static void scratch_parts(void* scratch, uint64_t frame_bytes, uint32_t** crc, uint64_t** q, float** sz) {
    uint8_t* s = static_cast<uint8_t*>(scratch);
    const uint64_t off = ((sda::crc_scratch_words(frame_bytes) * 4 + 255) / 256) * 256;
    *crc = reinterpret_cast<uint32_t*>(s);
    *q = reinterpret_cast<uint64_t*>(s + off);
    *sz = reinterpret_cast<float*>(s + off + 64);
}

sda_status sda_frame_encode(void* stream, const sda_frame_header* h, const void* x, int32_t x_dtype, uint8_t* out,
                            void* scratch, int32_t* err) {
    if (!h || !out || !scratch || h->n_dims > SDA_FRAME_MAX_DIMS || !frame_dtype_ok(h->dtype) || !quant_dtype_ok(x_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    const uint64_t count = sda_frame_elements(h);
    if (count > 0 && !x) return SDA_ERR_INVALID_ARGUMENT;
    uint8_t hdr[128];
    int n = 0;
    auto put = [&](uint64_t v, int bytes) {
        for (int i = 0; i < bytes; ++i) hdr[n++] = (uint8_t)(v >> (8 * i));
    };
    hdr[n++] = 'F'; hdr[n++] = 'A'; hdr[n++] = 'T'; hdr[n++] = 'N';   // frame.cpp:119-131
    put(h->version, 1);
    put(h->msg_type, 1);
    put(h->request_id, 8);
    put(h->layer, 2);
    put(h->head, 2);
    put(h->domain, 2);
    put(h->dtype, 1);
    put(h->n_dims, 4);
    for (uint32_t i = 0; i < h->n_dims; ++i) put(h->dims[i], 4);
    uint32_t* crc;
    uint64_t* q;
    float* sz;
    const uint64_t total = sda_frame_bytes(h);
    scratch_parts(scratch, total, &crc, &q, &sz);
    g_launches += 3;
    return from_cuda(sda::launch_frame_encode(x, x_dtype, (int64_t)count, h->dtype, hdr, n, out,
                                              sda_frame_payload_bytes(h), crc, q, sz, err,
                                              static_cast<cudaStream_t>(stream)));
}

sda_status sda_frame_parse_header(const uint8_t* b, uint64_t host_len, uint64_t frame_size, sda_frame_header* out) {
    if (!b || !out) return SDA_ERR_INVALID_ARGUMENT;
    if (frame_size < 29 || host_len < 25) return SDA_ERR_FRAME;                       // frame too short
    if (b[0] != 'F' || b[1] != 'A' || b[2] != 'T' || b[3] != 'N') return SDA_ERR_FRAME;   // bad magic
    auto get = [&](uint64_t pos, int bytes) {
        uint64_t v = 0;
        for (int i = 0; i < bytes; ++i) v |= (uint64_t)b[pos + i] << (8 * i);
        return v;
    };
    sda_frame_header h{};
    h.version = (uint8_t)get(4, 1);
    h.msg_type = (uint8_t)get(5, 1);
    h.request_id = get(6, 8);
    h.layer = (uint16_t)get(14, 2);
    h.head = (uint16_t)get(16, 2);
    h.domain = (uint16_t)get(18, 2);
    h.dtype = (uint8_t)get(20, 1);
    const uint64_t nd = get(21, 4);
    if (25 + 4 * nd + 4 > frame_size) return SDA_ERR_FRAME;                            // truncated
    if (nd > SDA_FRAME_MAX_DIMS) return SDA_ERR_UNSUPPORTED;
    if (host_len < 25 + 4 * nd) return SDA_ERR_INVALID_ARGUMENT;                       // pass the whole header
    h.n_dims = (uint32_t)nd;
    for (uint32_t i = 0; i < h.n_dims; ++i) h.dims[i] = (uint32_t)get(25 + 4 * i, 4);
    if (!frame_dtype_ok(h.dtype)) return SDA_ERR_FRAME;                                // unknown dtype
    if (frame_header_bytes(&h) + sda_frame_payload_bytes(&h) + 4 != frame_size) return SDA_ERR_FRAME;
    *out = h;
    return SDA_OK;
}

sda_status sda_frame_decode(void* stream, const uint8_t* frame, uint64_t frame_size, const sda_frame_header* h,
                            void* out, int32_t out_dtype, void* scratch, int32_t* err) {
    if (!h || !frame || !scratch || h->n_dims > SDA_FRAME_MAX_DIMS || !frame_dtype_ok(h->dtype) || !quant_dtype_ok(out_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if (sda_frame_bytes(h) != frame_size) return SDA_ERR_FRAME;
    const uint64_t count = sda_frame_elements(h);
    if (count > 0 && !out) return SDA_ERR_INVALID_ARGUMENT;
    uint32_t* crc;
    uint64_t* q;
    float* sz;
    scratch_parts(scratch, frame_size, &crc, &q, &sz);
    g_launches += 3;
    return from_cuda(sda::launch_frame_decode(frame, (int)frame_header_bytes(h), sda_frame_payload_bytes(h),
                                              (int64_t)count, h->dtype, out, out_dtype, crc, sz, err,
                                              static_cast<cudaStream_t>(stream)));
}

sda_status sda_crc32(void* stream, const uint8_t* bytes, uint64_t len, void* scratch, uint8_t* out4) {
    if ((!bytes && len) || !scratch || !out4) return SDA_ERR_INVALID_ARGUMENT;
    uint32_t* crc;
    uint64_t* q;
    float* sz;
    scratch_parts(scratch, len, &crc, &q, &sz);
    g_launches += 2;
    return from_cuda(sda::launch_crc32(bytes, len, crc, out4, static_cast<cudaStream_t>(stream)));
}

int32_t sda_default_splits(int64_t n_batch, int32_t q_heads, int64_t q_rows, int64_t kv_cap) {
    if (n_batch <= 0 || q_heads <= 0 || q_rows <= 0 || kv_cap <= 0) return 1;
    if (q_rows >= 64) {
        // prefill (tcgen05 kernel, one CTA per SM per 256 query rows x split): minimise
        //   ceil(waves) * (KV tiles per split + 4)  +  splits * merge cost
        // in units of one CTA's 128-key tile time (~1.86 us): each CTA pays ~4 tiles of pipeline
        // fill and epilogue, and every extra split is another (O', stats) set for K3 to read
        // (~0.022 tile-times per 256-row unit at ~3.3 TB/s). C3: 1 split (K2 493 us + K3 ~15 us)
        // instead of 4 (480 + 51 us); C5's prefill chunk: 2.
        const int64_t units = ((q_rows + 255) / 256) * q_heads * n_batch;
        const int64_t tiles = (kv_cap + 127) / 128;
        const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(8, tiles / 4));
        const double sms = (double)sda::device_sms();
        int32_t best = 1;
        double best_cost = 1e300;
        for (int64_t s = 1; s <= max_s; ++s) {
            const double waves = std::ceil((double)(units * s) / sms);
            const double cost = waves * ((double)((tiles + s - 1) / s) + 4.0) + (double)s * 0.022 * (double)units;
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = (int32_t)s;
            }
        }
        return best;
    }
    // Decode is HBM-bound and every CTA streams the same number of keys, so the last partial
    // wave of the grid runs the memory pipe at a fraction of its width: pick the split count
    // (>= 2 tiles of 128 keys per split) whose grid fills whole waves best, among grids of at
    // least 2 and at most ~12 waves (beyond that more splits only add partials and per-CTA
    // overhead); ties go to fewer splits (C2: 13 splits = 4.99 waves of 148 x 9 CTAs).
    const int64_t ctas = n_batch * q_heads * q_rows;
    const int64_t slots = (int64_t)sda::device_sms() * sda::k2_decode_ctas_per_sm();
    const int64_t max_by_len = std::max<int64_t>(1, kv_cap / 256);
    const int64_t s_max = std::min<int64_t>(max_by_len, SDA_MAX_SOURCES);   // K3 merges <= 64 sources
    int64_t best = 1;
    double best_eff = -1.0;
    for (int64_t s = 1; s <= s_max; ++s) {
        const double waves = (double)(s * ctas) / (double)slots;
        if (waves > 12.0 && best_eff > 0.0) break;
        if (waves < 2.0 && s < s_max) continue;
        const double eff = waves / std::ceil(waves);
        if (eff > best_eff + 1e-3) {
            best_eff = eff;
            best = s;
        }
    }
    return (int32_t)best;
}

int32_t sda_default_splits_gqa(int64_t n_batch, int32_t q_heads, int32_t kv_heads, int64_t q_rows, int64_t kv_cap,
                               int32_t head_dim) {
    if (n_batch <= 0 || q_heads <= 0 || kv_heads <= 0 || q_rows <= 0 || kv_cap <= 0) return 1;
    const int64_t G = q_heads / kv_heads;
    if (head_dim == 128 && G > 1 && G * q_rows <= 128 && q_rows < 64) {
        // grouped tensor-core decode: one CTA per SM (209 KB of SMEM), one per (request, kv
        // head, split); every CTA pays a pipeline fill / drain of ~2.6 KV tiles' time, so
        // minimise  waves * (tiles per split + 2.6)  (C5: 4 splits, 6.9 waves -- 16 % faster
        // than 37 splits = 64 exact waves of 14-tile CTAs; tools/gqa_bench.py)
        const int64_t units = n_batch * kv_heads;
        const int64_t tiles = (kv_cap + 127) / 128;
        const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(64, tiles / 4));
        int32_t best = 1;
        double best_cost = 1e300;
        for (int64_t s = 1; s <= max_s; ++s) {
            const double waves = std::ceil((double)(units * s) / (double)sda::device_sms());
            const double cost = waves * ((double)((tiles + s - 1) / s) + 2.6);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = (int32_t)s;
            }
        }
        return best;
    }
    if (head_dim == 128 && q_rows >= 64) {
        // prefill rows on the tensor-core form: one split runs stream-K (persistent groups of
        // n_qpairs CTAs over the linear tile order, k2_prefill_tc.cu): ~tiles / CTA + ~8 tiles of
        // segment fill / drain, x1.09 measured against the split grid's per-tile cost (static
        // ranges wait for the slowest SM; C3 471 vs 482 us, 27 heads 419 vs 512 us) -- against
        // the split grid's waves x (tiles per split + 4) + merge cost for S >= 2 (C5's prefill
        // chunk, 1024 CTAs = 6.9 full waves at S = 2, stays on the split grid: 3.60 vs 3.86 ms)
        const int64_t qpairs = (q_rows + 255) / 256;
        const int64_t units = qpairs * q_heads * n_batch;
        const int64_t tiles = (kv_cap + 127) / 128;
        const int64_t sms = sda::device_sms();
        const int64_t ctas = std::max<int64_t>(1, sms / qpairs) * qpairs;
        const double sk = qpairs <= sms ? 1.09 * ((double)(units * tiles) / (double)ctas + 8.0) : 1e300;
        const int64_t max_s = std::max<int64_t>(2, std::min<int64_t>(8, tiles / 4));
        int32_t best = 1;
        double best_cost = sk;
        for (int64_t s2 = 2; s2 <= max_s; ++s2) {
            const double waves = std::ceil((double)(units * s2) / (double)sms);
            const double cost = waves * ((double)((tiles + s2 - 1) / s2) + 4.0) + (double)s2 * 0.022 * (double)units;
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = (int32_t)s2;
            }
        }
        return best;
    }
    return sda_default_splits(n_batch, q_heads, q_rows, kv_cap);
}

size_t sda_prefill_workspace_bytes(int64_t n_batch, int32_t q_heads, int32_t kv_heads, int64_t q_rows, int64_t kv_cap,
                                   int32_t head_dim, int32_t q_dtype, int32_t kv_dtype) {
    if (n_batch <= 0 || q_rows <= 0 || kv_cap <= 0 || q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads != 0)
        return 0;
    sda::K2Params p{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, kv_cap, n_batch, q_rows, q_heads, kv_heads, 1,
                    0.f, 0, 0};
    if (!sda::k2_prefill_tc_eligible(p, head_dim, q_dtype, kv_dtype) || sda::k2_gqa_tc_eligible(p, head_dim, q_dtype, kv_dtype))
        return 0;
    return sda::k2_prefill_sk_workspace_bytes(p);
}

sda_status sda_partial_attention(void* stream, const void* q, int32_t q_dtype, const void* k, const void* v,
                                 int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int64_t n_batch,
                                 int32_t q_heads, int32_t kv_heads, int64_t q_rows, int32_t head_dim,
                                 int32_t n_splits, float* out_o, float* out_stats) {
    return sda_partial_attention_ws(stream, q, q_dtype, k, v, kv_dtype, kv_cap, kv_len, n_batch, q_heads, kv_heads, q_rows,
                                    head_dim, n_splits, out_o, out_stats, nullptr, 0);
}

sda_status sda_partial_attention_ws(void* stream, const void* q, int32_t q_dtype, const void* k, const void* v,
                                    int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int64_t n_batch,
                                    int32_t q_heads, int32_t kv_heads, int64_t q_rows, int32_t head_dim,
                                    int32_t n_splits, float* out_o, float* out_stats, void* workspace,
                                    size_t workspace_bytes) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    if (!q || !k || !v || !out_o || !out_stats || !valid_dtype_f64(q_dtype) || !valid_dtype_f64(kv_dtype) ||
        !f64_pair_ok(q_dtype, kv_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if (!row_aligned(q, head_dim, q_dtype) || !row_aligned(k, head_dim, kv_dtype) || !row_aligned(v, head_dim, kv_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch < 0 || q_rows < 0 || kv_cap < 0 || q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads != 0 ||
        n_splits <= 0)
        return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch * q_rows > 65535 || q_heads > 65535 || n_splits > 65535) return SDA_ERR_UNSUPPORTED;
    if (n_batch == 0 || q_rows == 0) return SDA_OK;
    sda::K2Params p{q, k, v, kv_len, out_o, out_stats, kv_cap, n_batch, q_rows, q_heads, kv_heads, n_splits,
                    (float)(1.0 / std::sqrt((double)head_dim)), 0, 0};
    if (q_dtype == SDA_F64) {
        ++g_launches;
        return from_cuda(sda::launch_f64_path(2, &p, head_dim, n_batch, static_cast<cudaStream_t>(stream)));
    }
    p.sk_work = workspace;
    p.sk_work_bytes = workspace ? workspace_bytes : 0;
    ++g_launches;
    if (sda::k2_gqa_tc_eligible(p, head_dim, q_dtype, kv_dtype) && !env_flag("SDA_K2_SIMT") &&
        !env_flag("SDA_K2_GROUPED"))
        return from_cuda(sda::launch_k2_gqa_tc(p, static_cast<cudaStream_t>(stream)));
    if (sda::k2_prefill_tc_eligible(p, head_dim, q_dtype, kv_dtype) && !env_flag("SDA_K2_SIMT"))
        return from_cuda(sda::launch_k2_prefill_tc(p, static_cast<cudaStream_t>(stream)));
    return from_cuda(sda::launch_k2_decode(p, head_dim, q_dtype, kv_dtype, static_cast<cudaStream_t>(stream)));
}

sda_status sda_partial_attention_causal(void* stream, const void* q, int32_t q_dtype, const void* k, const void* v,
                                        int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int64_t n_batch,
                                        int32_t q_heads, int32_t kv_heads, int64_t q_rows, int32_t head_dim,
                                        int32_t n_splits, int64_t causal_offset, float* out_o, float* out_stats) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    if (!q || !k || !v || !out_o || !out_stats || !valid_dtype_f64(q_dtype) || !valid_dtype_f64(kv_dtype) ||
        !f64_pair_ok(q_dtype, kv_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if (!row_aligned(q, head_dim, q_dtype) || !row_aligned(k, head_dim, kv_dtype) || !row_aligned(v, head_dim, kv_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch < 0 || q_rows < 0 || kv_cap < 0 || q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads != 0 ||
        n_splits <= 0)
        return SDA_ERR_INVALID_ARGUMENT;
    if (n_batch * q_rows > 65535 || q_heads > 65535 || n_splits > 65535) return SDA_ERR_UNSUPPORTED;
    if (n_batch == 0 || q_rows == 0) return SDA_OK;
    sda::K2Params p{q, k, v, kv_len, out_o, out_stats, kv_cap, n_batch, q_rows, q_heads, kv_heads, n_splits,
                    (float)(1.0 / std::sqrt((double)head_dim)), 1, causal_offset};
    ++g_launches;
    if (q_dtype == SDA_F64)
        return from_cuda(sda::launch_f64_path(2, &p, head_dim, n_batch, static_cast<cudaStream_t>(stream)));
    // prefill-sized spans (bf16, d 128, >= 64 rows): the tensor-core kernel with per-row key limits
    if (q_rows >= 64 && sda::k2_prefill_tc_eligible(p, head_dim, q_dtype, kv_dtype) &&
        !sda::k2_gqa_tc_eligible(p, head_dim, q_dtype, kv_dtype) && !env_flag("SDA_K2_SIMT"))
        return from_cuda(sda::launch_k2_prefill_tc(p, static_cast<cudaStream_t>(stream)));
    return from_cuda(sda::launch_k2_decode(p, head_dim, q_dtype, kv_dtype, static_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------------------------------
// LL exchange (decode): K1 writes Q' into the destinations' receive slots, K2 reads it from its
// own slot and writes every split's record into the inquirer's slot, K3 merges the records --
// all epoch-tagged (ll_store / ll_load in common.cuh), no separate copy, fence or flag.
// ------------------------------------------------------------------------------------------
sda_status sda_ll_scramble_q(void* stream, const void* q, int32_t q_dtype, int32_t n_dest, int64_t b_per,
                             int32_t n_heads, int32_t head_dim, const void* keys, int64_t keys_batch_stride,
                             int32_t key_heads, void* const* ll_q, int32_t wire_dtype, const uint32_t* epoch) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim) || head_dim < 64) return SDA_ERR_UNSUPPORTED;
    if (!q || !keys || !ll_q || !epoch || n_dest <= 0 || n_dest > sda::kMaxPeers || b_per <= 0 || n_heads <= 0 ||
        key_heads <= 0 || n_heads % key_heads != 0 || !valid_dtype(q_dtype) || !valid_dtype(wire_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < n_dest; ++i)
        if (!ll_q[i]) return SDA_ERR_INVALID_ARGUMENT;
    sda::K1Params p{};
    p.x = q;
    p.keys = keys;
    p.keys_bstride = keys_batch_stride;
    p.rows = 1;
    p.out_rows_cap = 1;
    p.n_heads = n_heads;
    p.key_heads = key_heads;
    p.which = SDA_KEYS_KQ;
    p.x_batch_mod = b_per;
    for (int i = 0; i < n_dest; ++i) p.ll_out[i] = ll_q[i];
    p.epoch = epoch;
    ++g_launches;
    return from_cuda(sda::launch_k1(p, head_dim, q_dtype, wire_dtype, (int64_t)n_dest * b_per,
                                    static_cast<cudaStream_t>(stream)));
}

sda_status sda_ll_partial_attention(void* stream, const void* ll_q, int32_t wire_dtype, const void* k, const void* v,
                                    int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int32_t n_dest,
                                    int64_t b_per, int32_t q_heads, int32_t kv_heads, int32_t head_dim,
                                    int32_t n_splits, void* const* ll_rec, const uint32_t* epoch, void* gqa_work) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim) || head_dim < 64) return SDA_ERR_UNSUPPORTED;
    if (!ll_q || !k || !v || !ll_rec || !epoch || n_dest <= 0 || n_dest > sda::kMaxPeers || b_per <= 0 ||
        q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads != 0 || n_splits <= 0 || kv_cap < 0 ||
        !valid_dtype(wire_dtype) || !valid_dtype(kv_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < n_dest; ++i)
        if (!ll_rec[i]) return SDA_ERR_INVALID_ARGUMENT;
    const int64_t n_batch = (int64_t)n_dest * b_per;
    if (n_batch > 65535 || q_heads > 65535 || n_splits > 65535) return SDA_ERR_UNSUPPORTED;
    sda::K2Params p{ll_q, k, v, kv_len, nullptr, nullptr, kv_cap, n_batch, 1, q_heads, kv_heads, n_splits,
                    (float)(1.0 / std::sqrt((double)head_dim)), 0, 0};
    p.epoch = epoch;
    p.b_per = b_per;
    for (int i = 0; i < n_dest; ++i) p.ll_rec[i] = ll_rec[i];
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (gqa_work && sda::k2_gqa_tc_eligible(p, head_dim, wire_dtype, kv_dtype) && !env_flag("SDA_K2_SIMT")) {
        // GQA: unpack Q' out of its LL words (spins on the epoch), then the tensor-core GQA
        // kernel reads it through TMA and writes its split records in LL form
        g_launches += 2;
        cudaError_t e = sda::launch_ll_unpack_q(ll_q, n_batch * q_heads * head_dim, gqa_work, epoch, st);
        if (e != cudaSuccess) return from_cuda(e);
        p.q = gqa_work;
        return from_cuda(sda::launch_k2_gqa_tc(p, st));
    }
    ++g_launches;
    return from_cuda(sda::launch_k2_decode(p, head_dim, wire_dtype, kv_dtype, st));
}

sda_status sda_partial_attention_remote(void* stream, const void* q, int32_t q_dtype, const void* k, const void* v,
                                        int32_t kv_dtype, int64_t kv_cap, const int32_t* kv_len, int32_t n_dest,
                                        int64_t b_per, int32_t q_heads, int32_t kv_heads, int64_t q_rows,
                                        int32_t head_dim, float* const* rec_peer, int64_t rec_stride,
                                        uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* dest_counters,
                                        void* workspace, size_t workspace_bytes) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    if (!q || !k || !v || !rec_peer || !peer_flag || !epoch || !dest_counters || n_dest <= 0 ||
        n_dest > sda::kMaxPeers || b_per <= 0 || q_heads <= 0 || kv_heads <= 0 || q_heads % kv_heads != 0 ||
        q_rows <= 0 || !valid_dtype(q_dtype) || !valid_dtype(kv_dtype) || rec_stride < (int64_t)q_heads * q_rows * (head_dim + 2))
        return SDA_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < n_dest; ++i)
        if (!rec_peer[i] || !peer_flag[i]) return SDA_ERR_INVALID_ARGUMENT;
    const int64_t n_batch = (int64_t)n_dest * b_per;
    if (n_batch * q_rows > 65535 || q_heads > 65535) return SDA_ERR_UNSUPPORTED;
    sda::K2Params p{q, k, v, kv_len, nullptr, nullptr, kv_cap, n_batch, q_rows, q_heads, kv_heads, 1,
                    (float)(1.0 / std::sqrt((double)head_dim)), 0, 0};
    if (!sda::k2_prefill_tc_eligible(p, head_dim, q_dtype, kv_dtype) || (q_heads / kv_heads > 1 && q_rows < 64))
        return SDA_ERR_UNSUPPORTED;   // the tensor-core prefill form only (one split per request)
    p.remote_rec = 1;
    p.epoch = epoch;
    p.b_per = b_per;
    p.rec_stride = rec_stride;
    for (int i = 0; i < n_dest; ++i) {
        p.ll_rec[i] = rec_peer[i];
        p.peer_flag[i] = peer_flag[i];
    }
    p.dest_counters = dest_counters;
    p.sk_work = workspace;
    p.sk_work_bytes = workspace ? workspace_bytes : 0;
    ++g_launches;
    return from_cuda(sda::launch_k2_prefill_tc(p, static_cast<cudaStream_t>(stream)));
}

sda_status sda_ll_unscramble_merge(void* stream, const void* ll_rec, int32_t n_domains, int32_t n_splits,
                                   const void* keys, int64_t keys_batch_stride, int32_t key_heads, int64_t b_per,
                                   int32_t q_heads, int32_t head_dim, void* out, int32_t out_dtype, uint32_t* epoch,
                                   uint32_t* done_counter) {
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim) || head_dim < 64) return SDA_ERR_UNSUPPORTED;
    if (!ll_rec || !keys || !out || !epoch || !done_counter || n_domains <= 0 || n_splits <= 0 || b_per <= 0 ||
        q_heads <= 0 || key_heads <= 0 || q_heads % key_heads != 0 || !valid_dtype(out_dtype))
        return SDA_ERR_INVALID_ARGUMENT;
    if ((int64_t)n_domains * n_splits > SDA_MAX_SOURCES) return SDA_ERR_UNSUPPORTED;
    sda::K3Params p{};
    const int64_t row = (int64_t)q_heads * (head_dim + 2);   // logical floats per request
    const uint8_t* base = static_cast<const uint8_t*>(ll_rec);
    for (int w = 0; w < n_domains; ++w)
        for (int s = 0; s < n_splits; ++s) {
            const uint8_t* blk = base + 8 * ((int64_t)(w * n_splits + s) * b_per * row);
            p.src[w * n_splits + s] = {reinterpret_cast<const float*>(blk), reinterpret_cast<const float*>(blk),
                                       static_cast<const uint8_t*>(keys) + (int64_t)w * b_per * keys_batch_stride,
                                       nullptr, row};
        }
    p.n_src = n_domains * n_splits;
    p.keys_bstride = keys_batch_stride;
    p.key_heads = key_heads;
    p.n_batch = b_per;
    p.q_heads = q_heads;
    p.q_rows = 1;
    p.out = out;
    p.ll = 1;
    p.epoch = epoch;
    p.done_counter = done_counter;
    ++g_launches;
    return from_cuda(sda::launch_k3(p, head_dim, out_dtype, static_cast<cudaStream_t>(stream)));
}

sda_status sda_unscramble_merge_quant(void* stream, const sda_merge_source* sources, int32_t n_sources,
                                      int64_t keys_batch_stride, int32_t key_heads, int64_t pq_batch_stride,
                                      int64_t n_batch, int32_t q_heads, int64_t q_rows, int32_t head_dim, void* out,
                                      int32_t out_dtype, float* out_stats, int32_t* err_flag, int64_t out_batch_stride,
                                      int32_t quant_bits, uint64_t* scratch) {
    if (quant_bits < 2 || quant_bits > 8) return SDA_ERR_INVALID_ARGUMENT;
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (head_dim < 32 || !supported_dim(head_dim) || out_dtype == SDA_F64) return SDA_ERR_UNSUPPORTED;
    if (n_sources <= 0) return SDA_ERR_EMPTY_SHARDS;
    if (!sources || n_sources > SDA_MAX_SOURCES) return SDA_ERR_INVALID_ARGUMENT;
    int groups = 1;
    for (int i = 1; i < n_sources; ++i) groups += sources[i].keys != sources[i - 1].keys;
    if (q_rows > 1 && !scratch) return SDA_ERR_INVALID_ARGUMENT;
    return unscramble_merge_impl(stream, sources, n_sources, keys_batch_stride, key_heads, pq_batch_stride, n_batch,
                                 q_heads, q_rows, head_dim, out, out_dtype, out_stats, err_flag, out_batch_stride,
                                 quant_bits, groups, reinterpret_cast<unsigned long long*>(scratch));
}

sda_status sda_unscramble_merge(void* stream, const sda_merge_source* sources, int32_t n_sources,
                                int64_t keys_batch_stride, int32_t key_heads, int64_t pq_batch_stride,
                                int64_t n_batch, int32_t q_heads, int64_t q_rows, int32_t head_dim, void* out,
                                int32_t out_dtype, float* out_stats, int32_t* err_flag, int64_t out_batch_stride) {
    return unscramble_merge_impl(stream, sources, n_sources, keys_batch_stride, key_heads, pq_batch_stride, n_batch,
                                 q_heads, q_rows, head_dim, out, out_dtype, out_stats, err_flag, out_batch_stride, 0,
                                 0, nullptr);
}

static sda_status unscramble_merge_impl(void* stream, const sda_merge_source* sources, int32_t n_sources,
                                        int64_t keys_batch_stride, int32_t key_heads, int64_t pq_batch_stride,
                                        int64_t n_batch, int32_t q_heads, int64_t q_rows, int32_t head_dim, void* out,
                                        int32_t out_dtype, float* out_stats, int32_t* err_flag,
                                        int64_t out_batch_stride, int quant_bits, int n_groups,
                                        unsigned long long* qscratch) {
    if (n_sources <= 0) return SDA_ERR_EMPTY_SHARDS;  // attention.cpp:90
    if (n_sources > SDA_MAX_SOURCES || !sources) return SDA_ERR_INVALID_ARGUMENT;
    if (!pow2(head_dim)) return SDA_ERR_NOT_POW2;
    if (!supported_dim(head_dim)) return SDA_ERR_UNSUPPORTED;
    if (!out || !valid_dtype_f64(out_dtype) || n_batch < 0 || q_rows < 0 || q_heads <= 0) return SDA_ERR_INVALID_ARGUMENT;
    bool any_keys = false;
    for (int i = 0; i < n_sources; ++i) {
        if (!sources[i].o || !sources[i].stats) return SDA_ERR_INVALID_ARGUMENT;
        any_keys |= sources[i].keys != nullptr;
    }
    if (any_keys && (key_heads <= 0 || q_heads % key_heads != 0)) return SDA_ERR_INVALID_ARGUMENT;
    if (head_dim >= 32 && out_dtype != SDA_F64) {
        // the warp forms move a row as one d/32-element vector per lane: every O' and output row
        // must start on that vector's alignment (up to 16 bytes), every stats pair on 8 bytes --
        // so pointers and batch strides must keep them there (a packed record of q_heads * q_rows
        // * (d + 2) floats does whenever q_heads * q_rows is even)
        auto misaligned = [](const void* ptr, int64_t stride_elems, int64_t esz, int64_t align) {
            return (reinterpret_cast<uintptr_t>(ptr) % align) != 0 || ((stride_elems * esz) % align) != 0;
        };
        const int64_t vin = std::min<int64_t>(16, (head_dim / 32) * 4);
        const int64_t osz = out_dtype == SDA_BF16 ? 2 : 4, vout = std::min<int64_t>(16, (head_dim / 32) * osz);
        for (int i = 0; i < n_sources; ++i)
            if (misaligned(sources[i].o, sources[i].batch_stride, 4, vin) ||
                misaligned(sources[i].stats, sources[i].batch_stride, 4, 8))
                return SDA_ERR_INVALID_ARGUMENT;
        if (misaligned(out, out_batch_stride, osz, vout) || (out_stats && misaligned(out_stats, out_batch_stride, 4, 8)))
            return SDA_ERR_INVALID_ARGUMENT;
    }
    if (n_batch == 0 || q_rows == 0) return SDA_OK;
    sda::K3Params p{};
    for (int i = 0; i < n_sources; ++i)
        p.src[i] = {sources[i].o, sources[i].stats, static_cast<const uint8_t*>(sources[i].keys), sources[i].pq_inv,
                    sources[i].batch_stride};
    p.n_src = n_sources;
    p.keys_bstride = keys_batch_stride;
    p.key_heads = key_heads > 0 ? key_heads : q_heads;
    p.pq_bstride = pq_batch_stride;
    p.n_batch = n_batch;
    p.q_heads = q_heads;
    p.q_rows = q_rows;
    p.out = out;
    p.out_stats = out_stats;
    p.err = err_flag;
    p.out_bstride = out_batch_stride;
    p.quant_bits = quant_bits;
    p.n_groups = n_groups;
    p.qscratch = qscratch;
    g_launches += quant_bits > 0 && q_rows > 1 ? 2 : 1;
    if (out_dtype == SDA_F64)   // FP64 mode: f64 sources and stats, f64 key images
        return from_cuda(sda::launch_f64_path(3, &p, head_dim, n_batch, static_cast<cudaStream_t>(stream)));
    return from_cuda(sda::launch_k3(p, head_dim, out_dtype, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
