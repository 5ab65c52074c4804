// common.cuh -- small device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sdattn_internal.h"

#include <mutex>
#include <set>
#include <utility>

namespace sda {

// SM count of the current device (grid sizing and the split heuristics); 148 on B200, also the
// answer without a device (host-side callers of the heuristics)
inline int device_sms() {
    static int cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return 148;
    }
    if (!cache[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;
        }
        cache[dev] = n;
    }
    return cache[dev];
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device, so a process driving several GPUs must set it on each of them
inline cudaError_t ensure_smem_attr(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16-byte streaming load that bypasses L1 allocation (KV tiles are read once).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void bf16x2_to_f2(uint32_t w, float& a, float& b) {
    a = __uint_as_float(w << 16);
    b = __uint_as_float(w & 0xFFFF0000u);
}

__device__ __forceinline__ uint32_t f2_to_bf16x2(float a, float b) {
    __nv_bfloat162 t = __floats2bfloat162_rn(a, b);  // RNE, single rounding
    return *reinterpret_cast<uint32_t*>(&t);
}

// Load N consecutive elements (N multiple of 8) of T starting at p (16-byte aligned) into f32.
template <int N, typename T>
__device__ __forceinline__ void load_vec(const T* p, float* v);

template <int N>
__device__ __forceinline__ void load_vec(const __nv_bfloat16* p, float* v) {
    static_assert(N % 8 == 0, "");
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
        const uint4 w = *reinterpret_cast<const uint4*>(p + 8 * i);
        bf16x2_to_f2(w.x, v[8 * i + 0], v[8 * i + 1]);
        bf16x2_to_f2(w.y, v[8 * i + 2], v[8 * i + 3]);
        bf16x2_to_f2(w.z, v[8 * i + 4], v[8 * i + 5]);
        bf16x2_to_f2(w.w, v[8 * i + 6], v[8 * i + 7]);
    }
}

template <int N>
__device__ __forceinline__ void load_vec(const float* p, float* v) {
    static_assert(N % 4 == 0, "");
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
        const float4 w = *reinterpret_cast<const float4*>(p + 4 * i);
        v[4 * i + 0] = w.x; v[4 * i + 1] = w.y; v[4 * i + 2] = w.z; v[4 * i + 3] = w.w;
    }
}

template <int N, typename T>
__device__ __forceinline__ void store_vec(T* p, const float* v);

template <int N>
__device__ __forceinline__ void store_vec(__nv_bfloat16* p, const float* v) {
    static_assert(N % 8 == 0, "");
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
        uint4 w;
        w.x = f2_to_bf16x2(v[8 * i + 0], v[8 * i + 1]);
        w.y = f2_to_bf16x2(v[8 * i + 2], v[8 * i + 3]);
        w.z = f2_to_bf16x2(v[8 * i + 4], v[8 * i + 5]);
        w.w = f2_to_bf16x2(v[8 * i + 6], v[8 * i + 7]);
        *reinterpret_cast<uint4*>(p + 8 * i) = w;
    }
}

template <int N>
__device__ __forceinline__ void store_vec(float* p, const float* v) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i)
        *reinterpret_cast<float4*>(p + 4 * i) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}

// Eight consecutive elements kept in their storage format until they are consumed (halves the
// registers a bf16 load needs, so more loads can be in flight per thread).
template <typename T>
struct Raw8;

template <>
struct Raw8<__nv_bfloat16> {
    uint4 w;
    __device__ __forceinline__ void load(const __nv_bfloat16* p) { w = ld_stream(p); }
    __device__ __forceinline__ float get(int i) const {
        const uint32_t x = i < 2 ? w.x : i < 4 ? w.y : i < 6 ? w.z : w.w;
        return (i & 1) ? __uint_as_float(x & 0xFFFF0000u) : __uint_as_float(x << 16);
    }
};

template <>
struct Raw8<float> {
    uint4 a, b;
    __device__ __forceinline__ void load(const float* p) {
        a = ld_stream(p);
        b = ld_stream(p + 4);
    }
    __device__ __forceinline__ float get(int i) const {
        const uint4& t = i < 4 ? a : b;
        const int j = i & 3;
        return __uint_as_float(j == 0 ? t.x : j == 1 ? t.y : j == 2 ? t.z : t.w);
    }
};

// Four consecutive elements in storage format (the d = 4 decode rows of K2).
template <typename T>
struct Raw4;

template <>
struct Raw4<__nv_bfloat16> {
    uint2 w;
    __device__ __forceinline__ void load(const __nv_bfloat16* p) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(p));
    }
    __device__ __forceinline__ float get(int i) const {
        const uint32_t x = i < 2 ? w.x : w.y;
        return (i & 1) ? __uint_as_float(x & 0xFFFF0000u) : __uint_as_float(x << 16);
    }
};

template <>
struct Raw4<float> {
    uint4 a;
    __device__ __forceinline__ void load(const float* p) { a = ld_stream(p); }
    __device__ __forceinline__ float get(int i) const {
        return __uint_as_float(i == 0 ? a.x : i == 1 ? a.y : i == 2 ? a.z : a.w);
    }
};

// N consecutive elements (N a power of two >= 4; 8-byte aligned for bf16 N = 4) into f32: the
// small head dims (d = 4, 8, 16) of the reference's own model tests
template <int N>
__device__ __forceinline__ void load_vec_n(const float* p, float* v) {
    load_vec<N>(p, v);
}
template <int N>
__device__ __forceinline__ void load_vec_n(const __nv_bfloat16* p, float* v) {
    if constexpr (N % 8 == 0) {
        load_vec<N>(p, v);
    } else {
        static_assert(N == 4, "");
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        bf16x2_to_f2(w.x, v[0], v[1]);
        bf16x2_to_f2(w.y, v[2], v[3]);
    }
}

// Small-vector variants for N in {1, 2, 4, 8, 16, ...} f32 loads / any-typed stores.
template <int N>
__device__ __forceinline__ void load_vec_any(const float* p, float* v) {
    if constexpr (N % 4 == 0) {
        load_vec<N>(p, v);
    } else if constexpr (N == 2) {
        const float2 w = *reinterpret_cast<const float2*>(p);
        v[0] = w.x; v[1] = w.y;
    } else {
        v[0] = p[0];
    }
}

template <int N>
__device__ __forceinline__ void store_vec_any(float* p, const float* v) {
    if constexpr (N % 4 == 0) {
        store_vec<N>(p, v);
    } else if constexpr (N == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
        p[0] = v[0];
    }
}

template <int N>
__device__ __forceinline__ void store_vec_any(__nv_bfloat16* p, const float* v) {
    if constexpr (N % 8 == 0) {
        store_vec<N>(p, v);
    } else if constexpr (N == 4) {
        uint2 w;
        w.x = f2_to_bf16x2(v[0], v[1]);
        w.y = f2_to_bf16x2(v[2], v[3]);
        *reinterpret_cast<uint2*>(p) = w;
    } else if constexpr (N == 2) {
        *reinterpret_cast<uint32_t*>(p) = f2_to_bf16x2(v[0], v[1]);
    } else {
        p[0] = __float2bfloat16_rn(v[0]);
    }
}

// Raw (unnormalised) Walsh-Hadamard butterflies over a vector of E*LPR elements held by a
// group of LPR consecutive lanes, lane lg owning elements [lg*E, lg*E+E). The 1/sqrt(d)
// normalisation of fwht.cpp:24 is folded into the packed output factors.
template <int E, int LPR>
__device__ __forceinline__ void fwht_group(float* v, int lane) {
#pragma unroll
    for (int h = 1; h < E; h <<= 1) {
#pragma unroll
        for (int i = 0; i < E; ++i) {
            if ((i & h) == 0) {
                const float a = v[i], b = v[i + h];
                v[i] = a + b;
                v[i + h] = a - b;
            }
        }
    }
#pragma unroll
    for (int m = 1; m < LPR; m <<= 1) {
        // lower lane: v + o, upper lane: o - v -- one FFMA with sign +-1 (exact: the product by
        // +-1 is exact and the FMA rounds once, as the add / subtract does)
        const float sgn = (lane & m) ? -1.f : 1.f;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const float o = __shfl_xor_sync(0xffffffffu, v[i], m);
            v[i] = fmaf(sgn, v[i], o);
        }
    }
}

// Programmatic dependent launch (the LL decode chain K1 -> K2 -> K3): a kernel launched with
// pdl_launch may start once every CTA of its predecessor has called pdl_trigger (or exited), so
// it overlaps the predecessor's tail instead of waiting for the grid to drain; pdl_wait blocks
// until the predecessor grid has completed and its writes are visible (no-op without PDL).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename Kern, typename... Args>
inline cudaError_t pdl_launch_smem(Kern kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <typename Kern, typename... Args>
inline cudaError_t pdl_launch(Kern kernel, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    return pdl_launch_smem(kernel, grid, block, 0, st, args...);
}

// raise a peer's flag to the step epoch with a system-scope release store (the waiting side
// polls it with acquire loads: exchange.cu wait_kernel)
__device__ __forceinline__ void flag_raise(uint32_t* flag, uint32_t e) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(e) : "memory");
}

// LL ("low-latency") peer-memory format for the decode exchange: every 4-byte data word is
// stored next to the 4-byte step epoch, two (data, epoch) pairs per 16-byte store. An aligned
// 8-byte half is written as one unit, so a reader that polls its words until both epochs match
// sees the data without any fence or separate flag: one NVLink write latency per exchange
// instead of store + system fence + flag store + flag poll.
__device__ __forceinline__ void ll_store(void* p, uint32_t a, uint32_t b, uint32_t e) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(e), "r"(b), "r"(e)
                 : "memory");
}
// Spin budget of every peer-memory wait (LL words, exchange flags): a wait that sees nothing for
// g_spin_timeout_ns gives up instead of hanging or trapping -- it records SDA_ERR_TIMEOUT in
// g_spin_error (read and cleared by sda_spin_error) and returns, so the kernel runs to its end and
// the CUDA context survives; the host reads the flag and tears the exchange down. Without
// relocatable device code every translation unit has its own copy of both; the TUs that spin
// export spin_access_<tu> (SDA_SPIN_ACCESSOR), through which sda_set_spin_timeout_ns and
// sda_spin_error reach them all.
static __device__ unsigned long long g_spin_timeout_ns = 30000000000ull;   // 30 s default
static __device__ int g_spin_error = 0;

// host: set this TU's timeout (set != nullptr), read its error word (err), clear it (clear)
#define SDA_SPIN_ACCESSOR(name)                                                                   \
    cudaError_t name(const unsigned long long* set, int* err, int clear) {                        \
        cudaError_t e = cudaSuccess;                                                              \
        if (set) e = cudaMemcpyToSymbol(g_spin_timeout_ns, set, sizeof(*set));                    \
        if (e == cudaSuccess && err) e = cudaMemcpyFromSymbol(err, g_spin_error, sizeof(int));   \
        if (e == cudaSuccess && clear) {                                                          \
            const int z = 0;                                                                      \
            e = cudaMemcpyToSymbol(g_spin_error, &z, sizeof(z));                                  \
        }                                                                                         \
        return e;                                                                                 \
    }

// true once the spin that started at t0 has used up its budget (the error is recorded once)
__device__ __forceinline__ bool spin_expired(uint64_t t0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 <= *(volatile unsigned long long*)&g_spin_timeout_ns) return false;
    atomicCAS(&g_spin_error, 0, (int)SDA_ERR_TIMEOUT);
    return true;
}

// spin until both epochs of the 16-byte word at p equal e (or the spin budget is used up: the
// stale words are returned and g_spin_error is set)
__device__ __forceinline__ uint2 ll_load(const void* p, uint32_t e) {
    uint32_t a, fa, b, fb;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(fa), "=r"(b), "=r"(fb) : "l"(p) : "memory");
    if (fa != e || fb != e) {
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {
            asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(a), "=r"(fa), "=r"(b), "=r"(fb) : "l"(p) : "memory");
            if (spin_expired(t0)) break;
        } while (fa != e || fb != e);
    }
    return make_uint2(a, b);
}

__host__ __device__ __forceinline__ const uint8_t* scrambler_ptr(const void* keys, int64_t batch_stride,
                                                                 int64_t b, int kh, int d, int which) {
    return static_cast<const uint8_t*>(keys) + b * batch_stride + (int64_t)kh * SDA_KEYSET_HEAD_BYTES(d) +
           (int64_t)which * SDA_SCRAMBLER_BYTES(d);
}

}  // namespace sda
