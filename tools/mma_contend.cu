// mma_contend.cu -- tcgen05.mma rates for the K2 prefill's own operand forms, alone and next to the
// softmax's TMEM traffic. Per SM: one CTA, warp 0's elected lane issues ITERS groups of MMAs into
// TMEM columns 256..383 (M = 128, N = 128, K = 16, bf16 -> f32), timed with clock64 around the
// final commit; optional "softmax" warps 1-8 meanwhile stream tcgen05.ld 32x32b.x16 of columns
// 128..255 (the other S) and tcgen05.st of 64 columns back (P), as the prefill kernel's softmax
// groups do. Modes:
//   0 SS, B K-major        (S = Q K^T)
//   1 TS, B MN-major       (O += P V: P from TMEM, V [keys x d] as an MN-major B, SW128 blocks)
//   2 TS, B K-major
//   3 mixed: 8 SS (mode 0) then 8 TS MN-major (mode 1) per group -- a prefill tile's S and PV
// Contention 1: softmax-like TMEM ld/st (warps 1-8); 2: TMA-like bulk fills into shared memory
// (warp 9, 32 KB per ~1850 cycles, the prefill kernel's average K/V fill rate).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_25716_b200/csrc -o tools/_mma_contend tools/mma_contend.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "tc_util.cuh"

using namespace sda;

constexpr int ITERS = 256;
constexpr int BLK = 128 * 128;   // [128 x 64] bf16 SW128 block

template <int MODE, int CONTEND>
__global__ void __launch_bounds__(320, 1) contend_kernel(unsigned long long* cycles, unsigned* sink, const uint8_t* gsrc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* a = smem;                  // Q: [128 x 128] bf16 K-major = 2 blocks (32 KB)
    uint8_t* b = smem + 2 * BLK;        // K or V: [128 x 128] bf16 = 2 blocks (32 KB)
    uint8_t* land = smem + 4 * BLK;     // TMA-like landing area (32 KB), CONTEND == 2
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 6 * BLK);
    uint64_t* bar2 = bar + 2;
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
    volatile uint32_t* stop = slot + 1;
    for (int i = threadIdx.x; i < 4 * BLK / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        tc::mbar_init(bar, 1);
        tc::mbar_init(bar2, 1);
        tc::fence_mbar_init();
        *stop = 0u;
    }
    if (threadIdx.x < 32) tc::tmem_alloc<512>(slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        const bool leader = tc::elect_one();
        constexpr uint32_t ID_SS = tc::idesc_bf16_f32(128, 128, false, false);
        constexpr uint32_t ID_TS_MN = tc::idesc_bf16_f32(128, 128, false, true);
        constexpr uint32_t ID_TS_K = tc::idesc_bf16_f32(128, 128, false, false);
        const uint32_t sa = tc::smem_u32(a), sb = tc::smem_u32(b);
        tc::fence_proxy_async_smem();
        const unsigned long long t0 = clock64();
        for (int it = 0; it < ITERS; ++it) {
            if (MODE == 0 || MODE == 3) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t off = (k >> 2) * BLK + (k & 3) * 32;
                    const uint64_t da = tc::sw128_desc(sa + off, 16, 1024), db = tc::sw128_desc(sb + off, 16, 1024);
                    if (leader) tc::mma_bf16_ss(tmem + 256, da, db, ID_SS, 1u);
                }
            }
            if (MODE == 1 || MODE == 3) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {   // as the prefill kernel's issue_pv
                    const uint64_t db = tc::sw128_desc(sb + k * 2048, BLK, 1024);
                    if (leader) tc::mma_bf16_ts(tmem + 384, tmem + k * 8, db, ID_TS_MN, 1u);
                }
            }
            if (MODE == 2) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t off = (k >> 2) * BLK + (k & 3) * 32;
                    const uint64_t db = tc::sw128_desc(sb + off, 16, 1024);
                    if (leader) tc::mma_bf16_ts(tmem + 384, tmem + k * 8, db, ID_TS_K, 1u);
                }
            }
        }
        if (leader) tc::mma_commit(bar);
        tc::mbar_wait(bar, 0);
        const unsigned long long t1 = clock64();
        if (threadIdx.x == 0) {
            cycles[blockIdx.x] = t1 - t0;
            *stop = 1u;
        }
    } else if (CONTEND == 2 && warp == 9) {
        // TMA-like fills: 32 KB (a K and a V tile's worth per two Q tiles' step) per ~1850 cycles,
        // the prefill kernel's average fill rate at its measured period, as two 16 KB bulk copies
        uint32_t ph = 0;
        int64_t off = 0;
        while (*stop == 0u) {
            const long long t = clock64();
            if (tc::elect_one()) {
                tc::mbar_arrive_expect_tx(bar2, 2 * BLK);
                for (int c = 0; c < 2; ++c)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(tc::smem_u32(land + c * BLK)), "l"(gsrc + off + c * BLK), "r"(BLK), "r"(tc::smem_u32(bar2))
                                 : "memory");
            }
            __syncwarp();
            tc::mbar_wait(bar2, ph);
            ph ^= 1u;
            off = (off + 2 * BLK + (int64_t)blockIdx.x * 4096) % ((int64_t)256 << 20);
            while (clock64() - t < 1850) {}
        }
    } else if (CONTEND == 1 && warp >= 1 && warp <= 8) {
        // softmax-like TMEM traffic on the other S columns (128..255) of this warp's lane quarter
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        unsigned acc = 0;
        while (*stop == 0u) {
            uint32_t s[64];
#pragma unroll
            for (int c = 0; c < 4; ++c) tc::tmem_ld16(tmem + lane_off + 128 + ((warp >> 2) & 1) * 64 + c * 16, s + c * 16);
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 64; ++i) acc += s[i];
            uint32_t pk[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) pk[e] = s[e] ^ acc;
#pragma unroll
            for (int c = 0; c < 2; ++c) tc::tmem_st8(tmem + lane_off + 128 + ((warp >> 2) & 1) * 64 + c * 8, pk);
            tc::tmem_st_wait();
        }
        if (acc == 0x12345678u) sink[0] = acc;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}

template <int MODE, int CONTEND>
void run(int sms, const char* name, const uint8_t* gsrc) {
    unsigned long long* d;
    unsigned* sink;
    cudaMalloc(&d, sms * 8);
    cudaMalloc(&sink, 4);
    const int smem = 6 * BLK + 64;
    cudaFuncSetAttribute(contend_kernel<MODE, CONTEND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    contend_kernel<MODE, CONTEND><<<sms, 320, smem>>>(d, sink, gsrc);
    contend_kernel<MODE, CONTEND><<<sms, 320, smem>>>(d, sink, gsrc);
    cudaDeviceSynchronize();
    unsigned long long h[256];
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i] / sms;
    const int per = MODE == 3 ? 16 : 8;
    printf("%-34s %s: %6.1f cycles per MMA (nominal 64) (%s)\n", name, CONTEND == 1 ? "+ softmax TMEM ld/st" : CONTEND == 2 ? "+ TMA-like fills    " : "alone               ",
           avg / ((double)per * ITERS), cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* g;
    cudaMalloc(&g, ((size_t)256 << 20) + 4 * BLK);
    cudaMemset(g, 0, ((size_t)256 << 20) + 4 * BLK);
    run<0, 0>(sms, "SS, B K-major (S = Q K^T)", g);
    run<0, 1>(sms, "SS, B K-major (S = Q K^T)", g);
    run<0, 2>(sms, "SS, B K-major (S = Q K^T)", g);
    run<1, 0>(sms, "TS, B MN-major (O += P V)", g);
    run<1, 1>(sms, "TS, B MN-major (O += P V)", g);
    run<1, 2>(sms, "TS, B MN-major (O += P V)", g);
    run<2, 0>(sms, "TS, B K-major", g);
    run<2, 1>(sms, "TS, B K-major", g);
    run<3, 0>(sms, "8 SS + 8 TS MN-major", g);
    run<3, 1>(sms, "8 SS + 8 TS MN-major", g);
    run<3, 2>(sms, "8 SS + 8 TS MN-major", g);
    cudaFree(g);
    return 0;
}
