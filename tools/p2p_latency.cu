// p2p_latency.cu -- microbenchmark of NVLink peer-memory signalling on one box (single process,
// peer access enabled between GPUs 0..n-1). Measures what bounds the exchange of the decode step:
//   1. flag ping-pong between GPU 0 and GPU 1 (one-way latency of a release store + acquire poll)
//   2. pushing `bytes` to every peer + raising its flag, for several block counts and fence styles,
//      with every GPU pushing at once (the exchange pattern), timed with events per GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_p2p_latency tools/p2p_latency.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// role 0 starts: for i: raise remote = 2i+1, wait local >= 2i+2. role 1: wait local >= 2i+1, raise remote 2i+2
__global__ void pingpong(uint32_t* local, uint32_t* remote, int iters, int role) {
    for (int i = 0; i < iters; ++i) {
        if (role == 0) {
            st_rel(remote, 2 * i + 1);
            while ((int)(ld_acq(local) - (2 * i + 2)) < 0) {}
        } else {
            while ((int)(ld_acq(local) - (2 * i + 1)) < 0) {}
            st_rel(remote, 2 * i + 2);
        }
    }
}

struct PushArgs {
    const uint4* src;
    uint4* dst[8];
    uint32_t* flag[8];
    unsigned* done;
    int64_t n16;
    uint32_t epoch;
};

// mode 0: all threads __threadfence_system; mode 1: __syncthreads + thread 0 fence; mode 2: st.release
// of the counter without a separate fence (release is cumulative)
template <int MODE>
__global__ void push(PushArgs a) {
    const int peer = blockIdx.y;
    uint4* d = a.dst[peer];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n16; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = a.src[i];
    if (MODE == 0) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (MODE == 1) __threadfence_system();
        unsigned prev;
        if (MODE == 2)
            asm volatile("atom.add.acq_rel.sys.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&a.done[peer]) : "memory");
        else
            prev = atomicAdd(&a.done[peer], 1u);
        if (prev == gridDim.x - 1) {
            a.done[peer] = 0;
            __threadfence_system();
            st_rel(a.flag[peer], a.epoch);
        }
    }
}

__global__ void waitk(const uint32_t* flags, int n, uint32_t e) {
    if (threadIdx.x < n) while ((int)(ld_acq(flags + threadIdx.x) - e) < 0) {}
    __syncthreads();
}

int main(int argc, char** argv) {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
    if (n > 8) n = 8;
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i));
        for (int j = 0; j < n; ++j) if (j != i) CK(cudaDeviceEnablePeerAccess(j, 0));
    }
    std::vector<uint32_t*> flags(n);
    std::vector<unsigned*> done(n);
    std::vector<uint4*> src(n), rbuf(n);
    const int64_t bytes = 128 * 1024;   // one destination slot of the cfg2 decode Q' (16 req x 32 heads x 128 x bf16)
    std::vector<cudaStream_t> st(n);
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i));
        CK(cudaMalloc(&flags[i], 64 * 4));
        CK(cudaMemset(flags[i], 0, 64 * 4));
        CK(cudaMalloc(&done[i], 64 * 4));
        CK(cudaMemset(done[i], 0, 64 * 4));
        CK(cudaMalloc(&src[i], bytes));
        CK(cudaMalloc(&rbuf[i], bytes * n));
        CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    }
    // ---- 1. ping-pong
    {
        const int iters = 10000;
        cudaEvent_t e0, e1;
        CK(cudaSetDevice(0));
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaSetDevice(1));
        pingpong<<<1, 1, 0, st[1]>>>(flags[1], flags[0], iters, 1);
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(e0, st[0]));
        pingpong<<<1, 1, 0, st[0]>>>(flags[0], flags[1], iters, 0);
        CK(cudaEventRecord(e1, st[0]));
        CK(cudaDeviceSynchronize());
        CK(cudaSetDevice(1));
        CK(cudaDeviceSynchronize());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("ping-pong GPU0<->GPU1: %.2f us one-way (%d round trips)\n", ms * 1e3 / iters / 2, iters);
        for (int i = 0; i < 2; ++i) { CK(cudaSetDevice(i)); CK(cudaMemset(flags[i], 0, 64 * 4)); }
    }
    // ---- 2. all-to-all push of `bytes` per peer + flags, every GPU at once
    uint32_t epoch = 0;
    for (int mode = 0; mode < 3; ++mode) {
        for (int blocks : {1, 4, 16, 64}) {
            const int reps = 200;
            std::vector<cudaEvent_t> a(n), b(n);
            for (int i = 0; i < n; ++i) {
                CK(cudaSetDevice(i));
                CK(cudaEventCreate(&a[i]));
                CK(cudaEventCreate(&b[i]));
            }
            for (int r = -5; r < reps; ++r) {
                ++epoch;
                for (int i = 0; i < n; ++i) {
                    CK(cudaSetDevice(i));
                    if (r == 0) CK(cudaEventRecord(a[i], st[i]));
                    PushArgs p{};
                    p.src = src[i];
                    for (int j = 0; j < n; ++j) {
                        p.dst[j] = rbuf[j] + (int64_t)i * (bytes / 16);
                        p.flag[j] = flags[j] + i;
                    }
                    p.done = done[i];
                    p.n16 = bytes / 16;
                    p.epoch = epoch;
                    dim3 g(blocks, n);
                    if (mode == 0) push<0><<<g, 256, 0, st[i]>>>(p);
                    if (mode == 1) push<1><<<g, 256, 0, st[i]>>>(p);
                    if (mode == 2) push<2><<<g, 256, 0, st[i]>>>(p);
                    waitk<<<1, 32, 0, st[i]>>>(flags[i], n, epoch);
                    if (r == reps - 1) CK(cudaEventRecord(b[i], st[i]));
                }
            }
            float worst = 0;
            for (int i = 0; i < n; ++i) {
                CK(cudaSetDevice(i));
                CK(cudaDeviceSynchronize());
                float ms;
                CK(cudaEventElapsedTime(&ms, a[i], b[i]));
                if (ms > worst) worst = ms;
            }
            printf("push+wait %d GPUs, %lld B/peer, fence mode %d, %2d blocks/peer: %.2f us per exchange\n", n,
                   (long long)bytes, mode, blocks, worst * 1e3 / reps);
        }
    }
    return 0;
}
