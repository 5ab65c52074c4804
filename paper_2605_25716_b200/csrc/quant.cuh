// quant.cuh -- the affine min-max quantiser's device arithmetic (quant.cpp:26-67), shared by the
// quantise / dequantise kernels (quant.cu) and the kernels that quantise in their epilogue or
// input path (K1 sda_scramble_quant, K3 sda_unscramble_merge_quant). Bit-exact with the
// reference on the same input values: see quant.cu.
#pragma once
#include <cmath>
#include <type_traits>

#include "common.cuh"

namespace sda {

// order-preserving u64 key of a double (for atomicMin / atomicMax)
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

template <typename T>
__device__ __forceinline__ double to_d(T v) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
        return (double)__bfloat162float(v);
    else
        return (double)v;
}
template <typename T>
__device__ __forceinline__ T from_d(double v) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
        return __float2bfloat16_rn(__double2float_rn(v));
    else if constexpr (std::is_same<T, float>::value)
        return __double2float_rn(v);
    else
        return v;
}

struct QParams {
    double zero, scale, inv;
    uint32_t levels;
    bool constant;
};

// zero = (float)lo ; scale = (float)((hi - lo) / levels) ; inv = 1 / (double)scale
__device__ __forceinline__ QParams qparams_lohi(double lo, double hi, int bits) {
    QParams q;
    q.levels = (1u << bits) - 1u;
    const float zf = __double2float_rn(lo);
    const float sf = __double2float_rn(__ddiv_rn(__dsub_rn(hi, lo), (double)q.levels));
    q.zero = (double)zf;
    q.scale = (double)sf;
    q.constant = sf == 0.f;
    q.inv = q.constant ? 0.0 : __drcp_rn(q.scale);
    return q;
}

__device__ __forceinline__ uint32_t qcode(double v, const QParams& q) {
    if (q.constant) return 0u;
    double c = rint(__dmul_rn(__dsub_rn(v, q.zero), q.inv));
    c = c < 0.0 ? 0.0 : c;
    c = c > (double)q.levels ? (double)q.levels : c;
    return (uint32_t)c;
}

__device__ __forceinline__ double qvalue(uint32_t code, const QParams& q) {
    return __dadd_rn(__dmul_rn((double)code, q.scale), q.zero);
}


// min / max of tensor t from the order-preserving keys a min / max pass left in kmin / kmax
__device__ __forceinline__ QParams qparams(const unsigned long long* kmin, const unsigned long long* kmax, int64_t t,
                                           int bits) {
    return qparams_lohi(dkey_inv(kmin[t]), dkey_inv(kmax[t]), bits);
}

// dequantize(quantize_affine(v)) of one value
__device__ __forceinline__ double qround(double v, const QParams& q) { return qvalue(qcode(v, q), q); }

}  // namespace sda
