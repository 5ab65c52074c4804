// exchange.cu -- the SCR_Q / SCR_SHARD exchange over NVLink peer memory, without NCCL.
//
// Replaces the simulated point-to-point frames of the reference protocol (Simulator::send of
// SCR_Q, protocol.cpp:892-896, and SCR_SHARD, protocol.cpp:1097-1102) inside one NVSwitch box:
// every rank maps its peers' receive buffers (CUDA IPC) and pushes its payloads straight into
// them with 16-byte stores over NVLink, then raises a per-sender flag with a system-scope
// release store; the receiver's wait kernel spins (acquire loads) on its own flags. A step
// epoch kept in device memory makes the whole sequence replayable from a CUDA graph.
//
// Safety of buffer reuse comes from the protocol itself: a sender's next SCR_Q push into rank r
// happens only after it has received r's SCR_SHARD for the current step, which r sends only after
// its K2 has consumed the current Q'; likewise for the return buffers. A spin that does not see
// its flag within the spin budget (sda_set_spin_timeout_ns, default 30 s) gives up and records
// SDA_ERR_TIMEOUT for sda_spin_error instead of hanging the GPU or trapping the context.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace sda {

struct PushParams {
    const uint4* src[kMaxPeers];     // local payload for peer p
    uint4* dst[kMaxPeers];           // peer p's receive slot (mapped peer memory)
    uint32_t* flag[kMaxPeers];       // peer p's flag for this sender (mapped peer memory)
    int n_peers;
    int64_t n16;                     // payload size in 16-byte units (same for every peer)
    const uint32_t* epoch;           // local step epoch
    unsigned int* done;              // local per-peer block counters (zeroed, self-resetting)
    int fence_one;                   // 1: thread 0 fences after the CTA barrier instead of every thread
};

__global__ void step_epoch_kernel(uint32_t* epoch) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *epoch += 1;
}

// grid (blocks_per_peer, n_peers): copy, fence, last block of a peer raises that peer's flag.
__global__ void __launch_bounds__(256) push_kernel(const PushParams p) {
    const int peer = blockIdx.y;
    const uint4* __restrict__ s = p.src[peer];
    uint4* d = p.dst[peer];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n16; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
    if (!p.fence_one) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        // one fence after the barrier covers the whole CTA's stores (fence cumulativity)
        if (p.fence_one) __threadfence_system();
        const unsigned int prev = atomicAdd(&p.done[peer], 1u);
        if (prev == gridDim.x - 1) {
            p.done[peer] = 0;
            __threadfence_system();
            const uint32_t e = *p.epoch;
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.flag[peer]), "r"(e) : "memory");
        }
    }
}

// one block: thread i waits until flags[i] (raised by sender i) reaches this step's epoch
__global__ void wait_kernel(const uint32_t* flags, int n, const uint32_t* epoch) {
    const int i = threadIdx.x;
    if (i < n) {
        const uint32_t e = *epoch;
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
            if ((int32_t)(v - e) >= 0) break;
            if (spin_expired(t0)) break;   // a peer is gone: record SDA_ERR_TIMEOUT, do not hang
            __nanosleep(64);
        }
    }
    __syncthreads();
}

SDA_SPIN_ACCESSOR(spin_access_exchange)

__global__ void timestamp_kernel(uint64_t* dst) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *dst = t;
}

}  // namespace sda

namespace {
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
    static AddrRangeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddrRangeFn>(ptr);
    }
    return fn;
}
sda_status from_cuda_x(cudaError_t e) { return e == cudaSuccess ? SDA_OK : SDA_ERR_CUDA; }
}  // namespace

extern "C" {

sda_status sda_ipc_get_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return SDA_ERR_INVALID_ARGUMENT;
    AddrRangeFn fn = addr_range_fn();
    if (!fn) return SDA_ERR_CUDA;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return SDA_ERR_CUDA;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
    if (e != cudaSuccess) return SDA_ERR_CUDA;
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
    return SDA_OK;
}

sda_status sda_ipc_open_handle(const void* handle, uint64_t offset, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return SDA_ERR_INVALID_ARGUMENT;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return SDA_ERR_CUDA;
    *dev_ptr_out = static_cast<uint8_t*>(base) + offset;
    return SDA_OK;
}

sda_status sda_ipc_close_handle(void* dev_ptr, uint64_t offset) {
    if (!dev_ptr) return SDA_ERR_INVALID_ARGUMENT;
    return from_cuda_x(cudaIpcCloseMemHandle(static_cast<uint8_t*>(dev_ptr) - offset));
}

sda_status sda_exchange_epoch(void* stream, uint32_t* epoch) {
    if (!epoch) return SDA_ERR_INVALID_ARGUMENT;
    sda::count_launch();
    sda::step_epoch_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(epoch);
    return from_cuda_x(cudaGetLastError());
}

sda_status sda_exchange_push(void* stream, int32_t n_peers, const void* const* src, void* const* dst,
                             uint32_t* const* peer_flags, uint64_t bytes, const uint32_t* epoch, uint32_t* counters) {
    if (n_peers <= 0 || n_peers > sda::kMaxPeers || !src || !dst || !peer_flags || !epoch || !counters ||
        bytes % 16 != 0)
        return SDA_ERR_INVALID_ARGUMENT;
    sda::PushParams p{};
    for (int i = 0; i < n_peers; ++i) {
        p.src[i] = static_cast<const uint4*>(src[i]);
        p.dst[i] = static_cast<uint4*>(dst[i]);
        p.flag[i] = peer_flags[i];
    }
    p.n_peers = n_peers;
    p.n16 = (int64_t)(bytes / 16);
    p.epoch = epoch;
    p.done = counters;
    static const int max_blocks = [] {
        const char* e = getenv("SDA_PUSH_BLOCKS");   // tuning knob (tools/step_timeline.py)
        return e && atoi(e) > 0 ? atoi(e) : 16;
    }();
    static const int fence_one = [] {
        const char* e = getenv("SDA_PUSH_FENCE_ONE");   // tuning knob (tools/step_timeline.py)
        return e && atoi(e) > 0 ? 1 : 0;
    }();
    p.fence_one = fence_one;
    int blocks = (int)std::min<int64_t>(max_blocks, (p.n16 + 255) / 256);
    if (blocks < 1) blocks = 1;
    sda::count_launch();
    sda::push_kernel<<<dim3(blocks, n_peers), 256, 0, static_cast<cudaStream_t>(stream)>>>(p);
    return from_cuda_x(cudaGetLastError());
}

sda_status sda_exchange_wait(void* stream, const uint32_t* flags, int32_t n, const uint32_t* epoch) {
    if (!flags || !epoch || n <= 0 || n > 1024) return SDA_ERR_INVALID_ARGUMENT;
    sda::count_launch();
    sda::wait_kernel<<<1, ((n + 31) / 32) * 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, n, epoch);
    return from_cuda_x(cudaGetLastError());
}

// every translation unit whose kernels spin on peer memory (common.cuh SDA_SPIN_ACCESSOR)
static cudaError_t spin_access_all(const unsigned long long* set, int* err, int clear) {
    cudaError_t (*const tus[])(const unsigned long long*, int*, int) = {
        sda::spin_access_exchange, sda::spin_access_k2_decode, sda::spin_access_k3_merge};
    int worst = 0;
    for (auto fn : tus) {
        int v = 0;
        const cudaError_t e = fn(set, err ? &v : nullptr, clear);
        if (e != cudaSuccess) return e;
        if (v) worst = v;
    }
    if (err) *err = worst;
    return cudaSuccess;
}

sda_status sda_set_spin_timeout_ns(uint64_t ns) {
    if (ns == 0) return SDA_ERR_INVALID_ARGUMENT;
    const unsigned long long v = ns;
    return from_cuda_x(spin_access_all(&v, nullptr, 0));
}

sda_status sda_spin_error(int32_t* out, int32_t clear) {
    if (!out) return SDA_ERR_INVALID_ARGUMENT;
    int v = 0;
    const cudaError_t e = spin_access_all(nullptr, &v, clear);
    *out = v;
    return from_cuda_x(e);
}

sda_status sda_trace_timestamp(void* stream, uint64_t* dst) {
    if (!dst) return SDA_ERR_INVALID_ARGUMENT;
    sda::timestamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dst);
    return from_cuda_x(cudaGetLastError());
}

}  // extern "C"
