// pipe_bench.cu -- per-SM issue throughput of the instructions the prefill softmax is made of
// (MUFU.EX2, F2FP bf16x2 pack, FFMA2, FMNMX3, IMAD), 8 independent chains per thread, 16 warps
// per SM. Prints warp-instructions per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void __launch_bounds__(512) kern(float* out, float seed) {
    float a[8];
    uint32_t u[8];
    uint64_t d[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        a[k] = seed * (threadIdx.x + k) * 1e-7f - 1.f;
        u[k] = __float_as_uint(a[k]);
        asm("mov.b64 %0, {%1, %2};" : "=l"(d[k]) : "f"(a[k]), "f"(a[k] * 0.5f));
    }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
            if (OP == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %0;" : "+r"(u[k]) : "f"(a[k]));
            if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d[k]));
            if (OP == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(a[(k + 1) & 7]), "f"(a[(k + 2) & 7]));
            if (OP == 4) asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(u[k]) : "r"(u[(k + 1) & 7]));
            if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[k]));
            if (OP == 6) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(d[k]));
            if (OP == 7) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[k]));
            if (OP == 8) asm volatile("cvt.rn.f16x2.f32 %0, %1, %0;" : "+r"(u[k]) : "f"(a[k]));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float x, y;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(d[k]));
        s += a[k] + __uint_as_float(u[k]) + x + y;
    }
    if (s == 123.456f) out[0] = s;
}

int main() {
    int sms = 0, clk_khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, 4);
    const char* names[] = {"MUFU.EX2 (ex2.approx)", "F2FP (cvt.rn.bf16x2.f32)", "FFMA2 (fma.rn.f32x2)", "FMNMX3 (max.f32 x3)",
                           "IMAD (mad.lo.u32)", "FFMA (fma.rn.f32)", "FADD2 (add.rn.f32x2)",
                           "MUFU.EX2 f16x2", "F2FP f16x2 (cvt.rn.f16x2.f32)"};
    for (int op = 0; op < 9; ++op) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int blocks = sms * 4, threads = 512;   // 64 warps per SM
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (op) {
                case 0: kern<0><<<blocks, threads>>>(out, 1.f); break;
                case 1: kern<1><<<blocks, threads>>>(out, 1.f); break;
                case 2: kern<2><<<blocks, threads>>>(out, 1.f); break;
                case 3: kern<3><<<blocks, threads>>>(out, 1.f); break;
                case 4: kern<4><<<blocks, threads>>>(out, 1.f); break;
                case 5: kern<5><<<blocks, threads>>>(out, 1.f); break;
                case 6: kern<6><<<blocks, threads>>>(out, 1.f); break;
                case 7: kern<7><<<blocks, threads>>>(out, 1.f); break;
                case 8: kern<8><<<blocks, threads>>>(out, 1.f); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warp_instr = (double)blocks * threads / 32 * ITERS * 8;
        const double per_sm_per_ns = warp_instr / sms / (ms * 1e6);
        printf("%-26s %.3f warp-instr/ns/SM  (= %.2f per clock at %.0f MHz nominal)\n", names[op], per_sm_per_ns,
               per_sm_per_ns / (clk_khz * 1e-6), clk_khz * 1e-3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
