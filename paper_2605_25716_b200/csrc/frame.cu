// frame.cu -- the "FATN" wire frame on the device (SURVEY 8(f) "next" row 3): encode a device
// tensor into the reference's bit-exact frame and decode one back, so the scrambled tensors of
// the GPU path (SCR_Q, SCR_KV, SCR_SHARD) can leave and enter as reference-compatible bytes.
//
// Replaces encode_frame / decode_frame / payload_from_values / values_from_payload
// (frame.cpp:113-164, :166-236) for tensor frames (make_tensor_frame, frame.cpp:238-262).
// Layout, little-endian: "FATN" | version u8 | msg_type u8 | request_id u64 | layer u16 |
// head u16 | domain u16 | dtype u8 | dim_count u32 | dims u32... | payload | crc32 u32 over all
// bytes before it (CRC-32/IEEE, reflected, poly 0xEDB88320, frame.cpp:17-25, :78-83).
// Payload element encodings: f64 raw; f32 = (float)v; bf16 / f16 = round_to_format's RNE onto
// the target grid with overflow clamped to the largest finite value (float_format.cpp:23-37),
// then the bit pattern (float_format.cpp:60-95); quantN = quantize_affine codes + scale + zero
// point as f32 (quant.cu).
//
// CRC on the device, in parallel: the message is cut into 256-byte chunks whose raw CRCs
// (register starting at 0) are independent; raw CRC is linear over GF(2), so
//   raw(A || B) = Z^|B| raw(A) xor raw(B)       (Z^n: the 32x32 "feed n zero bytes" operator)
// and a power-of-two tree with Z^(256 * 2^k) per level combines them (zero chunks prepended to
// reach a power of two change nothing: zeros fed to a zero register stay zero). The standard
// conditioning is one more term: crc = ~(Z^N 0xFFFFFFFF xor raw(M)); the sub-chunk tail is fed
// byte by byte into the combined register. Z^n matrices are built on the host by squaring.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace sda {

constexpr int kCrcChunk = 256;       // bytes per independent chunk
constexpr int kMaxLevels = 40;       // tree levels (2^40 chunks)

struct Gf2Mat {
    uint32_t col[32];                // col[i] = operator applied to the single bit 1 << i
};

struct CrcPlan {
    Gf2Mat level[kMaxLevels];        // Z^(kCrcChunk * 2^k)
    uint32_t k_prefix;               // Z^P 0xFFFFFFFF, P = full-chunk prefix length
    int levels;                      // log2 of the padded chunk count
};

namespace {

__device__ __forceinline__ uint32_t gf2_apply(const Gf2Mat& m, uint32_t v) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
        if (v & (1u << i)) r ^= m.col[i];
    return r;
}

__device__ uint32_t g_crc_tables[4][256];   // slicing-by-4 tables (filled once)

__global__ void crc_tables_kernel() {
    const uint32_t i = threadIdx.x;
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    g_crc_tables[0][i] = c;
    __syncthreads();
    for (int t = 1; t < 4; ++t) {
        const uint32_t p = g_crc_tables[t - 1][i];
        g_crc_tables[t][i] = g_crc_tables[0][p & 0xFF] ^ (p >> 8);
        __syncthreads();
    }
}

// raw CRC (register from 0) of each full 256-byte chunk -> acc[pad + j]
__global__ void __launch_bounds__(256) crc_chunks_kernel(const uint8_t* __restrict__ msg, int64_t n_chunks,
                                                         uint32_t* acc, int64_t pad) {
    __shared__ uint32_t T[4][256];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) T[i >> 8][i & 255] = g_crc_tables[i >> 8][i & 255];
    __syncthreads();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_chunks; j += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t* p = msg + j * kCrcChunk;
        uint32_t c = 0;
        for (int w = 0; w < kCrcChunk; w += 16) {
            // bytes as LE u32 words (the frame's byte offsets are not 4-aligned: unaligned-safe)
            uint32_t v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                v[q] = (uint32_t)p[w + 4 * q] | ((uint32_t)p[w + 4 * q + 1] << 8) | ((uint32_t)p[w + 4 * q + 2] << 16) |
                       ((uint32_t)p[w + 4 * q + 3] << 24);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                c ^= v[q];
                c = T[3][c & 0xFF] ^ T[2][(c >> 8) & 0xFF] ^ T[1][(c >> 16) & 0xFF] ^ T[0][c >> 24];
            }
        }
        acc[pad + j] = c;
    }
}

// one block of 1024 threads: power-of-two tree over acc[0 .. 2^levels), then the conditioning
// term, the sub-chunk tail byte by byte, and the final inversion -> *crc_out (and, when
// `write_to` is set, the 4 LE bytes at write_to; when `check` is set, *err if they differ)
__global__ void __launch_bounds__(1024) crc_combine_kernel(uint32_t* acc, const CrcPlan plan, const uint8_t* tail,
                                                           int tail_len, uint8_t* write_to, const uint8_t* check,
                                                           int32_t* err, int32_t err_code) {
    __shared__ uint32_t sh[1024];
    const int64_t n = (int64_t)1 << plan.levels;
    const int T = (int)(n < 1024 ? n : 1024);
    const int64_t per = n / T;   // power of two
    int lvl = 0;
    uint32_t v = 0;
    if ((int)threadIdx.x < T) {
        // thread-local tree over its `per` consecutive chunks
        uint32_t* a = acc + (int64_t)threadIdx.x * per;
        for (int64_t w = 1; w < per; w <<= 1, ++lvl)
            for (int64_t i = 0; i + w < per; i += 2 * w) a[i] = gf2_apply(plan.level[lvl], a[i]) ^ a[i + w];
        v = a[0];
        sh[threadIdx.x] = v;
    }
    __syncthreads();
    for (int w = 1; w < T; w <<= 1, ++lvl) {
        if ((int)threadIdx.x < T && (threadIdx.x % (2 * w)) == 0)
            sh[threadIdx.x] = gf2_apply(plan.level[lvl], sh[threadIdx.x]) ^ sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        uint32_t c = plan.k_prefix ^ (plan.levels >= 0 && T > 0 ? sh[0] : 0u);
        for (int i = 0; i < tail_len; ++i) c = g_crc_tables[0][(c ^ tail[i]) & 0xFF] ^ (c >> 8);
        c = ~c;
        if (write_to)
            for (int i = 0; i < 4; ++i) write_to[i] = (uint8_t)(c >> (8 * i));
        if (check) {
            const uint32_t want = (uint32_t)check[0] | ((uint32_t)check[1] << 8) | ((uint32_t)check[2] << 16) |
                                  ((uint32_t)check[3] << 24);
            if (want != c && err) *err = err_code;
        }
    }
}

// ---- element encodings (float_format.cpp) ---------------------------------------------------
// round_spec: RNE onto a grid with `mbits` explicit mantissa bits and minimum normal exponent
// emin, +-inf and overflow clamped to +-max_finite, 0 / NaN unchanged
__device__ __forceinline__ double round_spec(double x, int mbits, int emin, double max_finite) {
    if (x == 0.0 || isnan(x)) return x;
    if (isinf(x)) return copysign(max_finite, x);
    const int e = ilogb(x);
    const int q = (e < emin ? emin : e) - mbits;
    const double quantum = ldexp(1.0, q);
    double y = rint(x / quantum) * quantum;   // x / quantum is exact (power of two)
    if (fabs(y) > max_finite) y = copysign(max_finite, y);
    return y;
}
__device__ __forceinline__ uint16_t bf16_bits(double x) {
    const double y = round_spec(x, 7, -126, 0x1.FEp127);
    return (uint16_t)(__float_as_uint((float)y) >> 16);   // exact: y is on the bf16 grid
}
__device__ __forceinline__ uint16_t f16_bits(double x) {
    const double y = round_spec(x, 10, -14, 65504.0);
    const uint16_t sign = signbit(y) ? 0x8000 : 0;
    if (y == 0.0) return sign;
    const double a = fabs(y);
    const int e = ilogb(a);
    if (e < -14) return sign | (uint16_t)rint(a * 0x1.0p24);   // subnormal
    return sign | (uint16_t)((e + 15) << 10) | (uint16_t)rint((ldexp(a, -e) - 1.0) * 1024.0);
}
__device__ __forceinline__ double from_f16_bits(uint16_t b) {
    const double sign = (b & 0x8000) ? -1.0 : 1.0;
    const int exp = (b >> 10) & 0x1F, mant = b & 0x3FF;
    if (exp == 0) return sign * ldexp((double)mant, -24);
    if (exp == 31) return mant == 0 ? sign * INFINITY : __longlong_as_double(0x7FF8000000000000ll);
    return sign * ldexp(1.0 + (double)mant / 1024.0, exp - 15);
}

template <typename T>
__device__ __forceinline__ double ld(const T* x, int64_t i) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
        return (double)__bfloat162float(x[i]);
    else
        return (double)x[i];
}

struct HeaderBytes {
    uint8_t b[128];
    int len;
};

// payload of a float wire dtype + the header (block 0)
template <typename T>
__global__ void __launch_bounds__(256) frame_encode_kernel(const T* __restrict__ x, int64_t count, int wire,
                                                           const HeaderBytes hdr, uint8_t* out) {
    if (blockIdx.x == 0 && (int)threadIdx.x < hdr.len) out[threadIdx.x] = hdr.b[threadIdx.x];
    uint8_t* pl = out + hdr.len;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = ld(x, i);
        switch (wire) {
            case 0: {   // f64
                const uint64_t u = (uint64_t)__double_as_longlong(v);
                for (int k = 0; k < 8; ++k) pl[8 * i + k] = (uint8_t)(u >> (8 * k));
                break;
            }
            case 1: {   // f32
                const uint32_t u = __float_as_uint((float)v);
                for (int k = 0; k < 4; ++k) pl[4 * i + k] = (uint8_t)(u >> (8 * k));
                break;
            }
            default: {   // bf16 / f16
                const uint16_t u = wire == 2 ? bf16_bits(v) : f16_bits(v);
                pl[2 * i] = (uint8_t)u;
                pl[2 * i + 1] = (uint8_t)(u >> 8);
            }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) frame_decode_kernel(const uint8_t* __restrict__ pl, int64_t count, int wire,
                                                           T* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double v;
        switch (wire) {
            case 0: {
                uint64_t u = 0;
                for (int k = 0; k < 8; ++k) u |= (uint64_t)pl[8 * i + k] << (8 * k);
                v = __longlong_as_double((long long)u);
                break;
            }
            case 1: {
                uint32_t u = 0;
                for (int k = 0; k < 4; ++k) u |= (uint32_t)pl[4 * i + k] << (8 * k);
                v = (double)__uint_as_float(u);
                break;
            }
            case 2: v = (double)__uint_as_float(((uint32_t)pl[2 * i] | ((uint32_t)pl[2 * i + 1] << 8)) << 16); break;
            default: v = from_f16_bits((uint16_t)(pl[2 * i] | (pl[2 * i + 1] << 8)));
        }
        if constexpr (std::is_same<T, __nv_bfloat16>::value)
            out[i] = __float2bfloat16_rn(__double2float_rn(v));
        else if constexpr (std::is_same<T, float>::value)
            out[i] = __double2float_rn(v);
        else
            out[i] = v;
    }
}

// the quantN trailer: scale and zero point as LE f32 after the codes
__global__ void quant_trailer_kernel(const float* sz, uint8_t* dst) {
    const int i = threadIdx.x;   // 8 threads
    if (i < 8) dst[i] = (uint8_t)(__float_as_uint(sz[i >> 2]) >> (8 * (i & 3)));
}
__global__ void quant_trailer_read_kernel(const uint8_t* src, float* sz) {
    if (threadIdx.x < 2) {
        uint32_t u = 0;
        for (int k = 0; k < 4; ++k) u |= (uint32_t)src[4 * threadIdx.x + k] << (8 * k);
        sz[threadIdx.x] = __uint_as_float(u);
    }
}

// ---- host: GF(2) operators --------------------------------------------------------------
Gf2Mat gf2_mul(const Gf2Mat& a, const Gf2Mat& b) {   // a o b
    Gf2Mat r;
    for (int i = 0; i < 32; ++i) {
        uint32_t v = b.col[i], o = 0;
        for (int k = 0; k < 32; ++k)
            if (v & (1u << k)) o ^= a.col[k];
        r.col[i] = o;
    }
    return r;
}
uint32_t gf2_apply_h(const Gf2Mat& m, uint32_t v) {
    uint32_t r = 0;
    for (int i = 0; i < 32; ++i)
        if (v & (1u << i)) r ^= m.col[i];
    return r;
}
Gf2Mat zero_byte_op() {   // register after feeding one zero byte
    Gf2Mat m;
    for (int i = 0; i < 32; ++i) {
        uint32_t c = 1u << i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
        m.col[i] = c;
    }
    return m;
}
Gf2Mat zeros_op(uint64_t n) {   // Z^n by square-and-multiply
    Gf2Mat r;
    for (int i = 0; i < 32; ++i) r.col[i] = 1u << i;
    Gf2Mat p = zero_byte_op();
    while (n) {
        if (n & 1) r = gf2_mul(p, r);
        p = gf2_mul(p, p);
        n >>= 1;
    }
    return r;
}

std::atomic<bool> tables_ready[64] = {};   // per device

cudaError_t crc_launch(const uint8_t* msg, uint64_t len, uint32_t* scratch, uint8_t* write_to, const uint8_t* check,
                       int32_t* err, int32_t err_code, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (!tables_ready[dev]) {
        crc_tables_kernel<<<1, 256, 0, st>>>();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        tables_ready[dev] = true;
    }
    const int64_t n_chunks = (int64_t)(len / kCrcChunk);
    int levels = 0;
    while (((int64_t)1 << levels) < n_chunks) ++levels;
    const int64_t n2 = (int64_t)1 << levels;
    static Gf2Mat level_ops[kMaxLevels];   // Z^(256 * 2^k), built once per process
    static std::once_flag once;
    std::call_once(once, [] {
        Gf2Mat m = zeros_op(kCrcChunk);
        for (int k = 0; k < kMaxLevels; ++k) {
            level_ops[k] = m;
            m = gf2_mul(m, m);
        }
    });
    CrcPlan plan;   // per call (kernel parameter): reentrant
    memcpy(plan.level, level_ops, sizeof(level_ops));
    plan.levels = n_chunks > 0 ? levels : 0;
    plan.k_prefix = gf2_apply_h(zeros_op((uint64_t)n_chunks * kCrcChunk), 0xFFFFFFFFu);
    cudaError_t e = cudaMemsetAsync(scratch, 0, (size_t)n2 * 4, st);
    if (e != cudaSuccess) return e;
    if (n_chunks > 0) {
        const int64_t blocks = std::min<int64_t>((n_chunks + 255) / 256, (int64_t)device_sms() * 8);
        crc_chunks_kernel<<<(unsigned)blocks, 256, 0, st>>>(msg, n_chunks, scratch, n2 - n_chunks);
    }
    crc_combine_kernel<<<1, 1024, 0, st>>>(scratch, plan, msg + (uint64_t)n_chunks * kCrcChunk,
                                           (int)(len - (uint64_t)n_chunks * kCrcChunk), write_to, check, err, err_code);
    return cudaGetLastError();
}

}  // namespace

uint64_t crc_scratch_words(uint64_t len) {
    const int64_t n_chunks = (int64_t)(len / kCrcChunk);
    int64_t n2 = 1;
    while (n2 < n_chunks) n2 <<= 1;
    return (uint64_t)n2;
}

cudaError_t launch_crc32(const uint8_t* msg, uint64_t len, uint32_t* scratch, uint8_t* out4, cudaStream_t st) {
    return crc_launch(msg, len, scratch, out4, nullptr, nullptr, 0, st);
}

cudaError_t launch_frame_encode(const void* x, int x_dt, int64_t count, int wire, const uint8_t* header, int hlen,
                                uint8_t* out, uint64_t payload_bytes, uint32_t* crc_scratch, uint64_t* q_scratch,
                                float* q_sz, int32_t* err, cudaStream_t st) {
    HeaderBytes h;
    memcpy(h.b, header, hlen);
    h.len = hlen;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)device_sms() * 8));
    cudaError_t e = cudaSuccess;
    if (wire <= 3) {
        switch (x_dt) {
            case SDA_F32: frame_encode_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(x), count, wire, h, out); break;
            case SDA_F64: frame_encode_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(x), count, wire, h, out); break;
            default:
                frame_encode_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), count, wire,
                                                                          h, out);
        }
        e = cudaGetLastError();
    } else {   // quantN: header, codes (quant.cu), scale + zero point
        frame_encode_kernel<float><<<1, 256, 0, st>>>(nullptr, 0, 1, h, out);
        const int bits = wire - 16;
        const uint64_t code_bytes = ((uint64_t)count * bits + 7) / 8;
        if (count > 0) {
            e = cudaMemsetAsync(out + hlen, 0, code_bytes, st);
            if (e == cudaSuccess)
                e = launch_quantize(x, x_dt, 1, count, bits, out + hlen, (int64_t)code_bytes, q_sz, q_sz + 1,
                                    reinterpret_cast<unsigned long long*>(q_scratch), err, st);
        } else {
            e = cudaMemsetAsync(q_sz, 0, 8, st);
        }
        if (e != cudaSuccess) return e;
        quant_trailer_kernel<<<1, 32, 0, st>>>(q_sz, out + hlen + code_bytes);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    return crc_launch(out, (uint64_t)hlen + payload_bytes, crc_scratch, out + hlen + payload_bytes, nullptr, nullptr, 0,
                      st);
}

// x <- round_to_format(x, fmt) in place (float_format.cpp:26-58; the float-format wire_round of
// model.cpp:339-348 / protocol.cpp:179): fmt 0 f64 (no-op), 1 f32, 2 bf16, 3 f16
template <typename T>
__global__ void __launch_bounds__(256) wire_round_kernel(T* x, int64_t n, int fmt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = (double)x[i];
        double y;
        if (fmt == 1) y = (double)(float)v;
        else if (fmt == 2) y = round_spec(v, 7, -126, 0x1.FEp127);
        else y = round_spec(v, 10, -14, 65504.0);
        x[i] = (T)y;
    }
}

cudaError_t launch_wire_round(void* x, int dt, int64_t n, int fmt, cudaStream_t st) {
    if (fmt == 0 || n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)device_sms() * 8));
    if (dt == SDA_F32) wire_round_kernel<float><<<blocks, 256, 0, st>>>(static_cast<float*>(x), n, fmt);
    else wire_round_kernel<double><<<blocks, 256, 0, st>>>(static_cast<double*>(x), n, fmt);
    return cudaGetLastError();
}

cudaError_t launch_frame_decode(const uint8_t* frame, int hlen, uint64_t payload_bytes, int64_t count, int wire,
                                void* out, int out_dt, uint32_t* crc_scratch, float* q_sz, int32_t* err,
                                cudaStream_t st) {
    cudaError_t e = crc_launch(frame, (uint64_t)hlen + payload_bytes, crc_scratch, nullptr, frame + hlen + payload_bytes,
                               err, SDA_ERR_FRAME, st);
    if (e != cudaSuccess || count == 0) return e;
    const uint8_t* pl = frame + hlen;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)device_sms() * 8));
    if (wire <= 3) {
        switch (out_dt) {
            case SDA_F32: frame_decode_kernel<float><<<blocks, 256, 0, st>>>(pl, count, wire, static_cast<float*>(out)); break;
            case SDA_F64: frame_decode_kernel<double><<<blocks, 256, 0, st>>>(pl, count, wire, static_cast<double*>(out)); break;
            default: frame_decode_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(pl, count, wire, static_cast<__nv_bfloat16*>(out));
        }
        return cudaGetLastError();
    }
    const int bits = wire - 16;
    const uint64_t code_bytes = ((uint64_t)count * bits + 7) / 8;
    quant_trailer_read_kernel<<<1, 32, 0, st>>>(pl + code_bytes, q_sz);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_dequantize(pl, (int64_t)code_bytes, q_sz, q_sz + 1, 1, count, bits, out, out_dt, st);
}

}  // namespace sda
