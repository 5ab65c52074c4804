// read_bw.cu -- streaming-read ceiling of this GPU's HBM: a grid-stride 16-byte-load reduction over
// 2 GiB (no writes but one word per block), several grid sizes and loads in flight per thread.
// Context for K2 decode's 7.1-7.3 TB/s. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_read_bw tools/read_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) rd(const uint4* __restrict__ p, int64_t n, unsigned* out) {
    unsigned acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + (int64_t)u * blockDim.x;
            if (j < n) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
            else v[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

int main() {
    const int64_t bytes = 2ll << 30, n = bytes / 16;
    uint4* p;
    unsigned* o;
    cudaMalloc(&p, bytes);
    cudaMalloc(&o, 1 << 20);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int waves : {1, 2, 4, 8}) {
        for (int u : {2, 4, 8}) {
            const int grid = sms * 8 * waves;
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(a);
                if (u == 2) rd<2><<<grid, 256>>>(p, n, o);
                if (u == 4) rd<4><<<grid, 256>>>(p, n, o);
                if (u == 8) rd<8><<<grid, 256>>>(p, n, o);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("grid %6d (8 CTAs x %d per SM) U=%d: %7.1f us  %.3f TB/s\n", grid, waves, u, best * 1e3, bytes / best / 1e9);
        }
    }
    return 0;
}
