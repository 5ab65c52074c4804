// quant.cu -- the quantised wire (SURVEY 8(f) "next" row 4): per-tensor affine min-max
// quantisation with 2..8-bit codes packed LSB-first, its inverse, and the quantise->dequantise
// round trip the reference applies to Q', K', V' and O' on a quantised wire.
//
// Replaces quantize_affine / dequantize (quant.cpp:26-67) as used by wire_round
// (model.cpp:338-341) and the protocol's gen_quant_bits frames (protocol.hpp:25-26). Bit-exact
// with the reference on the same input values: the min / max are exact, and the scale, zero
// point, codes and dequantised values follow the reference's f64 operation sequence with
// explicitly rounded f64 ops (no contraction):
//   zero = (float)lo ; scale = (float)((hi - lo) / levels) ; inv = 1 / (double)scale
//   code = clamp(rint(((double)v - (double)zero) * inv), 0, levels)     (nearbyint = RNE)
//   value = (double)code * (double)scale + (double)zero
// A constant tensor has scale 0 and all codes 0. Non-finite input sets *err (the reference
// throws std::invalid_argument).
//
// HBM-bound byte work: a min/max pass (one read) and a pack pass (one read, bits/8 B written per
// element). Packing is race-free without atomics: 8 consecutive elements fill exactly `bits`
// bytes, so each thread owns one group of 8.
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "quant.cuh"

namespace sda {

namespace {

// grid (x, n_tensors): per-tensor min / max of the finite values; any non-finite value -> *err
template <typename T>
__global__ void __launch_bounds__(256) qminmax_kernel(const T* __restrict__ x, int64_t count, unsigned long long* kmin,
                                                      unsigned long long* kmax, int32_t* err) {
    const int64_t t = blockIdx.y;
    const T* xs = x + t * count;
    double lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = to_d(xs[i]);
        if (!isfinite(v)) bad = true;
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    if (bad && err) atomicExch(err, (int32_t)SDA_ERR_INVALID_ARGUMENT);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, m));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, m));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(kmin + t, dkey(lo));
        atomicMax(kmax + t, dkey(hi));
    }
}

// grid (x, n_tensors): thread = group of 8 elements -> `bits` bytes of codes
template <typename T>
__global__ void __launch_bounds__(256) qpack_kernel(const T* __restrict__ x, int64_t count, int bits,
                                                    const unsigned long long* kmin, const unsigned long long* kmax,
                                                    uint8_t* codes, int64_t codes_stride, float* scale_out,
                                                    float* zero_out) {
    const int64_t t = blockIdx.y;
    const QParams q = qparams(kmin, kmax, t, bits);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (scale_out) scale_out[t] = (float)q.scale;
        if (zero_out) zero_out[t] = (float)q.zero;
    }
    const T* xs = x + t * count;
    uint8_t* cs = codes + t * codes_stride;
    const int64_t groups = (count + 7) / 8, nbytes = (count * bits + 7) / 8;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        uint64_t acc = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int64_t i = g * 8 + e;
            if (i < count) acc |= (uint64_t)qcode(to_d(xs[i]), q) << (e * bits);
        }
        const int64_t b0 = g * bits;
        for (int k = 0; k < bits && b0 + k < nbytes; ++k) cs[b0 + k] = (uint8_t)(acc >> (8 * k));
    }
}

template <typename T>
__global__ void __launch_bounds__(256) qdequant_kernel(const uint8_t* __restrict__ codes, int64_t codes_stride,
                                                       const float* __restrict__ scale, const float* __restrict__ zero,
                                                       int64_t count, int bits, T* out) {
    const int64_t t = blockIdx.y;
    const uint8_t* cs = codes + t * codes_stride;
    QParams q;
    q.scale = (double)scale[t];
    q.zero = (double)zero[t];
    const uint32_t mask = (1u << bits) - 1u;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bit = i * bits;
        const uint32_t w = (uint32_t)cs[bit >> 3] | ((bit + bits > ((bit >> 3) + 1) * 8) ? (uint32_t)cs[(bit >> 3) + 1] << 8 : 0u);
        out[t * count + i] = from_d<T>(qvalue((w >> (bit & 7)) & mask, q));
    }
}

// quantise -> dequantise in place (wire emulation, model.cpp:338-341)
template <typename T>
__global__ void __launch_bounds__(256) qroundtrip_kernel(T* x, int64_t count, int bits, const unsigned long long* kmin,
                                                         const unsigned long long* kmax) {
    const int64_t t = blockIdx.y;
    const QParams q = qparams(kmin, kmax, t, bits);
    T* xs = x + t * count;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        xs[i] = from_d<T>(qvalue(qcode(to_d(xs[i]), q), q));
}

unsigned blocks_for(int64_t work) {
    const int64_t b = (work + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 1184 ? 1184 : b));   // <= 8 CTAs per SM per tensor row
}

template <typename T>
cudaError_t minmax_t(const void* x, int64_t n, int64_t count, unsigned long long* scratch, int32_t* err, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(scratch, 0xFF, n * 8, st);                    // min keys
    if (e == cudaSuccess) e = cudaMemsetAsync(scratch + n, 0x00, n * 8, st);       // max keys
    if (e != cudaSuccess) return e;
    qminmax_kernel<T><<<dim3(blocks_for(count), (unsigned)n), 256, 0, st>>>(static_cast<const T*>(x), count, scratch,
                                                                            scratch + n, err);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const void* x, int dt, int64_t n, int64_t count, int bits, uint8_t* codes,
                            int64_t codes_stride, float* scale, float* zero, unsigned long long* scratch, int32_t* err,
                            cudaStream_t st) {
    cudaError_t e;
    const dim3 g(blocks_for((count + 7) / 8), (unsigned)n);
    switch (dt) {
        case SDA_F32:
            if ((e = minmax_t<float>(x, n, count, scratch, err, st)) != cudaSuccess) return e;
            qpack_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(x), count, bits, scratch, scratch + n,
                                                   codes, codes_stride, scale, zero);
            break;
        case SDA_F64:
            if ((e = minmax_t<double>(x, n, count, scratch, err, st)) != cudaSuccess) return e;
            qpack_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(x), count, bits, scratch, scratch + n,
                                                    codes, codes_stride, scale, zero);
            break;
        case SDA_BF16:
            if ((e = minmax_t<__nv_bfloat16>(x, n, count, scratch, err, st)) != cudaSuccess) return e;
            qpack_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), count, bits, scratch,
                                                           scratch + n, codes, codes_stride, scale, zero);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint8_t* codes, int64_t codes_stride, const float* scale, const float* zero,
                              int64_t n, int64_t count, int bits, void* out, int dt, cudaStream_t st) {
    const dim3 g(blocks_for(count), (unsigned)n);
    switch (dt) {
        case SDA_F32: qdequant_kernel<float><<<g, 256, 0, st>>>(codes, codes_stride, scale, zero, count, bits, static_cast<float*>(out)); break;
        case SDA_F64: qdequant_kernel<double><<<g, 256, 0, st>>>(codes, codes_stride, scale, zero, count, bits, static_cast<double*>(out)); break;
        case SDA_BF16:
            qdequant_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(codes, codes_stride, scale, zero, count, bits,
                                                              static_cast<__nv_bfloat16*>(out));
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_quant_roundtrip(void* x, int dt, int64_t n, int64_t count, int bits, unsigned long long* scratch,
                                   int32_t* err, cudaStream_t st) {
    cudaError_t e;
    const dim3 g(blocks_for(count), (unsigned)n);
    switch (dt) {
        case SDA_F32:
            if ((e = minmax_t<float>(x, n, count, scratch, err, st)) != cudaSuccess) return e;
            qroundtrip_kernel<float><<<g, 256, 0, st>>>(static_cast<float*>(x), count, bits, scratch, scratch + n);
            break;
        case SDA_F64:
            if ((e = minmax_t<double>(x, n, count, scratch, err, st)) != cudaSuccess) return e;
            qroundtrip_kernel<double><<<g, 256, 0, st>>>(static_cast<double*>(x), count, bits, scratch, scratch + n);
            break;
        case SDA_BF16:
            if ((e = minmax_t<__nv_bfloat16>(x, n, count, scratch, err, st)) != cudaSuccess) return e;
            qroundtrip_kernel<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<__nv_bfloat16*>(x), count, bits, scratch,
                                                                scratch + n);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace sda
