// mma_bench.cu -- tcgen05.mma (kind::f16, bf16 in, f32 accumulate, cta_group::1, M = 128) issue
// throughput per SM as a function of N, A from SMEM (SS) and from TMEM (TS): how many dense bf16
// FLOP per SM-clock each instruction shape delivers (the shape question behind the prefill
// kernel's tile choice). One CTA per SM, one elected thread issues ITERS x 4 MMAs (K = 64 per
// group) into one accumulator; timed with clock64 around the commit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_25716_b200/csrc -o tools/_mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_util.cuh"

using namespace sda;

constexpr int ITERS = 512;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_kernel(unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* a = smem;                 // [128 x 64] bf16 SW128 K-major (16 KB)
    uint8_t* b = smem + 16384;         // [N x 64] bf16 SW128 K-major
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 256 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        tc::mbar_init(bar, 1);
        tc::fence_mbar_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc<512>(slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x < 32) {
        const bool leader = tc::elect_one();
        constexpr uint32_t IDESC = tc::idesc_bf16_f32(128, N, false, false);
        const uint32_t sa = tc::smem_u32(a), sb = tc::smem_u32(b);
        tc::fence_proxy_async_smem();
        const unsigned long long t0 = clock64();
        for (int it = 0; it < ITERS; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t db = tc::sw128_desc(sb + k * 32, 16, 1024);
                if (TS) {
                    if (leader) tc::mma_bf16_ts(tmem + 256, tmem + k * 8, db, IDESC, 1u);   // A: 128 x 16 bf16 from TMEM
                } else {
                    const uint64_t da = tc::sw128_desc(sa + k * 32, 16, 1024);
                    if (leader) tc::mma_bf16_ss(tmem + 256, da, db, IDESC, 1u);
                }
            }
        }
        if (leader) tc::mma_commit(bar);
        tc::mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(int sms) {
    unsigned long long* d;
    cudaMalloc(&d, sms * 8);
    const int smem = 16384 + 256 * 128 + 64;
    cudaFuncSetAttribute(mma_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_kernel<N, TS><<<sms, 128, smem>>>(d);
    mma_kernel<N, TS><<<sms, 128, smem>>>(d);
    cudaDeviceSynchronize();
    unsigned long long h[256];
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i] / sms;
    const double flop = 2.0 * 128 * N * 16 * 4 * ITERS;
    printf("M=128 N=%3d K=16 %s: %6.1f cycles per MMA, %7.0f FLOP/clk/SM (%s)\n", N, TS ? "TS (A in TMEM)" : "SS            ",
           avg / (4.0 * ITERS), flop / avg, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, false>(sms);
    run<128, false>(sms);
    run<256, false>(sms);
    run<64, true>(sms);
    run<128, true>(sms);
    run<256, true>(sms);
    return 0;
}
