// k1_tc.cu -- K1 on the 5th-generation tensor cores: scramble + token permutation as a
// tcgen05 GEMM with a signed-diagonal-times-±1 B operand, cp.async row gather into swizzled
// SMEM, TMEM accumulators and a TMA store.
//
// Replaces apply_phi / apply_phi_inv_t + permute_rows_gather (scrambler.cpp:42-85,
// permutation.cpp:58-67) for the large, bf16 case: the context owner's KV shipping
// (protocol.cpp:993-1001) and prefill Q (protocol.cpp:885-891).
//
// With R = 1/sqrt(d) and the raw Sylvester matrix, x phi = ((x o s1) M) o (s2 R) where
//   M[i][n] = (-1)^popcount(P1[i] & P2^{-1}[n])
// (P1 and P2 collapse into the sign pattern), and the inverse-transpose uses
// 1/s1 and R/s2 with the same M. M is exact in bf16; diag(s1) M is split into bf16 hi + lo
// (16 significant bits), so D = x B_hi + x B_lo in f32 is accurate to ~2^-17 before the single
// RNE rounding to bf16 -- the same numerics as the f64 reference up to that rounding.
//
// Per CTA (persistent, one per SM, a contiguous run of 128-row tiles of one or more
// (request, head) slabs), warp-specialised, 9 warps:
//   warps 4-7 (loaders) : cp.async 16-byte chunks of the gathered input rows perm[r] straight
//                         into a SWIZZLE_128B K-major A stage (4 stages); completion is signalled
//                         with cp.async.mbarrier.arrive.noinc on the stage's `full` barrier;
//   warp 8     (MMA)    : the elected lane issues 2 x d/16 tcgen05.mma (M=128, N=d, K=16) into one of
//                         two TMEM accumulators; tcgen05.commit frees the A stage and hands the
//                         accumulator to the epilogue;
//   warps 0-3 (epilogue): tcgen05.ld -> bf16 -> swizzled SMEM -> TMA tensor
//                         store (a tile's output rows are contiguous in the cache), masked plain
//                         stores on a partial tile; they also (re)build B when the key set changes.
// B folds both diagonals: B[n][i] = (-1)^popc(P1[i] & P2inv[n]) * s1^{+-1}[i] * s2^{+-1}[n] R,
// split into bf16 hi + lo (16 significant bits), so x needs no prologue and the epilogue no
// scaling: D = x B_hi^T + x B_lo^T in f32 (~2^-17 relative) -> one RNE rounding to bf16.
// HBM-bound: 2 x 128 x d x 2 B per tile vs 2 x 128 x d x d x 2 flop (128 flop/B at d=128, below
// the 258 flop/B ridge).
#include "common.cuh"
#include "tc_util.cuh"

#include <algorithm>
#include <cstdlib>

namespace sda {

// One scramble job (the arguments of one sda_scramble call); a launch runs up to kK1Jobs of them
// back to back in one persistent grid (e.g. the span's K, V and Q of a prefill step).
struct K1TcJob {
    const __nv_bfloat16* x;
    __nv_bfloat16* out;
    const uint8_t* keys;
    const uint32_t* perm;
    int64_t keys_bstride;
    int64_t perm_bstride;
    int64_t rows;
    int64_t out_rows_cap;
    int64_t out_row_offset;
    int n_heads;
    int key_heads;
    int which;
    int inv_t;
    int64_t tiles_per_slab;
    int64_t x_batch_mod;
};
constexpr int kK1Jobs = 16;

struct K1TcParams {
    K1TcJob job[kK1Jobs];
    int64_t job_tile0[kK1Jobs + 1];   // first global tile of each job (prefix sums)
    int n_jobs;
    int64_t total_tiles;
    int64_t tiles_per_cta;
    int trace;
    // remote jobs (out in a peer's memory): once all of a job's tiles are stored, the CTA that
    // completes it raises *peer_flag[job] = *epoch (system-scope release); null = local job
    uint32_t* peer_flag[kK1Jobs];
    uint32_t* job_counters;           // [kK1Jobs] zeroed, self-resetting
    const uint32_t* epoch;
};

// Debug timeline (SDA_K1TC_TRACE=1): clock64 stamps per CTA -- [0] start, [1] first B built, and
// per tile it < 10: [2+5it] loader issues the gather, [3+5it] MMA warp sees the stage full,
// [4+5it] MMAs issued, [5+5it] epilogue sees the accumulator, [6+5it] its store issued.
// Read back with sda_debug_k1tc_trace (tools/k1_trace.py).
constexpr int kK1TraceSlots = 64;
__device__ unsigned long long g_k1tc_trace[256][kK1TraceSlots];

struct K1OutMaps {                    // one TMA store map per job (kernel parameter, 64-byte aligned)
    CUtensorMap m[kK1Jobs];
};

template <int D>
struct K1TcShape {
    static constexpr int TILE = 128;
    static constexpr int STAGES = 4;
    static constexpr int ROW_BYTES = D * 2;
    static constexpr int TILE_BYTES = TILE * ROW_BYTES;      // one bf16 tile (A stage / out staging)
    static constexpr int KB = D / 64;                        // 64-wide K (or N) blocks
    static constexpr int BLK_BYTES = TILE * 128;             // one [128 x 64] swizzled block of A
    static constexpr int BBLK_BYTES = D * 128;               // one [D x 64] swizzled block of B
    static constexpr int OFF_A = 0;                          // STAGES x A
    static constexpr int OFF_BHI = OFF_A + STAGES * TILE_BYTES;
    static constexpr int OFF_BLO = OFF_BHI + D * D * 2;
    static constexpr int OFF_OUT = OFF_BLO + D * D * 2;      // output staging
    static constexpr int OFF_BAR = OFF_OUT + TILE_BYTES;
    static constexpr int NBAR = 2 * STAGES + 4 + 2;          // full, empty, tmem_full, tmem_empty, bfree, bready
    static constexpr int OFF_KT = OFF_BAR + 8 * NBAR + 16;   // key tables of the B being built
    static constexpr int SMEM = OFF_KT + D * (4 + 4 + 2 + 2);
    static constexpr uint32_t TMEM_COLS = 2 * D;
#ifndef SDA_K1_LOADER_WARPS
#define SDA_K1_LOADER_WARPS 8   // measured: 4 -> 8 warps 391 -> 368 us on the 2 GiB fill, 12 no better
#endif
    static constexpr int LOADER_WARPS = SDA_K1_LOADER_WARPS;
    static constexpr int LOADERS = 32 * LOADER_WARPS;       // warps 4 .. 4 + LOADER_WARPS - 1
    static constexpr int MMA_WARP = 4 + LOADER_WARPS;
    static constexpr int THREADS = 32 * (MMA_WARP + 1);
};

template <int D>
__global__ void __launch_bounds__(K1TcShape<D>::THREADS, 1) k1_tc_kernel(const K1TcParams p, const __grid_constant__ K1OutMaps maps) {
    using S = K1TcShape<D>;
    constexpr int ST = S::STAGES;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* const a_base = smem + S::OFF_A;
    uint8_t* const b_hi = smem + S::OFF_BHI;
    uint8_t* const b_lo = smem + S::OFF_BLO;
    uint8_t* const ostg = smem + S::OFF_OUT;
    uint64_t* const full = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
    uint64_t* const empty = full + ST;
    uint64_t* const tfull = empty + ST;
    uint64_t* const tempty = tfull + 2;
    uint64_t* const bfree = tempty + 2;
    uint64_t* const bready = bfree + 1;
    uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(bready + 1);

    const int tid = threadIdx.x, warp = tid >> 5;
    auto stamp = [&](int slot) {
        if (p.trace && (tid & 31) == 0 && slot < kK1TraceSlots && blockIdx.x < 256)
            g_k1tc_trace[blockIdx.x][slot] = clock64();
    };
    const int64_t first = (int64_t)blockIdx.x * p.tiles_per_cta;
    const int64_t last = min(first + p.tiles_per_cta, p.total_tiles);
    if (first >= last) return;
    const int64_t ntiles = last - first;
    // global tile id -> (job, tile id within the job)
    auto job_of = [&](int64_t id) -> int {
        int j = 0;
        while (j + 1 < p.n_jobs && id >= p.job_tile0[j + 1]) ++j;
        return j;
    };

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < ST; ++s) {
            tc::mbar_init(&full[s], S::LOADERS);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(&tfull[0], 1);
        tc::mbar_init(&tfull[1], 1);
        tc::mbar_init(&tempty[0], 128);
        tc::mbar_init(&tempty[1], 128);
        tc::mbar_init(bfree, 1);
        tc::mbar_init(bready, 128);
        tc::fence_mbar_init();
        for (int j = 0; j < p.n_jobs; ++j) tc::prefetch_tmap(&maps.m[j]);
    }
    if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp == 0) stamp(0);

    auto tile_rows = [&](const K1TcJob& jb, int64_t lid) -> int {
        const int64_t rem = jb.rows - (lid % jb.tiles_per_slab) * S::TILE;
        return (int)(rem < S::TILE ? rem : (int64_t)S::TILE);
    };
    // key slab (request, key head) of a tile, tagged with its job: B is rebuilt when it changes
    auto kslab_of = [&](int64_t id) -> int64_t {
        const int j = job_of(id);
        const K1TcJob& jb = p.job[j];
        const int64_t slab = (id - p.job_tile0[j]) / jb.tiles_per_slab;
        const int G = jb.n_heads / jb.key_heads;
        return ((int64_t)j << 48) + (slab / jb.n_heads) * jb.key_heads + (slab % jb.n_heads) / G;
    };
    constexpr int CPR = D / 8;   // 16-byte chunks per row

    if (warp >= 4 && warp < S::MMA_WARP) {
        // ------------------------------------------------------------------ loaders
        const int lt = tid - 128;                  // 0 .. LOADERS - 1
        constexpr int RSTEP = S::LOADERS / CPR, NR = S::TILE / RSTEP;
        const int c = lt % CPR, r0 = lt / CPR;
        // source rows of a tile for this thread (-1: past the segment end); fetched two tiles
        // ahead so the perm-load latency overlaps earlier tiles' copies
        auto fetch_src = [&](int64_t it, int32_t* src) {
            const int64_t id = first + it;
            const K1TcJob& jb = p.job[job_of(id)];
            const int64_t lid = id - p.job_tile0[job_of(id)];
            const int64_t slab = lid / jb.tiles_per_slab, t = lid % jb.tiles_per_slab;
            const int nrows = tile_rows(jb, lid);
            const uint32_t* pm = jb.perm ? jb.perm + (slab / jb.n_heads) * jb.perm_bstride + t * S::TILE : nullptr;
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const int r = r0 + k * RSTEP;
                src[k] = r < nrows ? (pm ? (int32_t)__ldg(pm + r) : (int32_t)(t * S::TILE + r)) : -1;
            }
        };
        // three index buffers used in rotation with static names (the loop is unrolled by 3): tile
        // it's indices were loaded two tiles earlier and nothing copies a register whose load may
        // still be in flight (a cur = nxt move would stall on that load and cut the look-ahead to
        // one tile -- the perm loads cost ~12 % of K1's bandwidth that way, tools/k1_bench.py)
        int32_t ia[NR], ib[NR], ic[NR];
        auto tile = [&](int64_t it, const int32_t (&use)[NR], int32_t (&fetch)[NR]) {
            const int st = (int)(it % ST);
            if (it + 2 < ntiles) fetch_src(it + 2, fetch);
            if (it >= ST) tc::mbar_wait(&empty[st], (uint32_t)(((it / ST) - 1) & 1));
            if (warp == 4 && it < 10) stamp(2 + 5 * (int)it);
            const int jj = job_of(first + it);
            const K1TcJob& jb = p.job[jj];
            const int64_t slab = (first + it - p.job_tile0[jj]) / jb.tiles_per_slab;
            const int H = jb.n_heads;
            const int64_t xslab = jb.x_batch_mod > 0 ? ((slab / H) % jb.x_batch_mod) * H + slab % H : slab;
            const __nv_bfloat16* xs = jb.x + xslab * jb.rows * D + c * 8;
            uint8_t* a = a_base + st * S::TILE_BYTES + (c >> 3) * S::BLK_BYTES;
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const int r = r0 + k * RSTEP;
                if (use[k] >= 0) tc::cp_async16(a + tc::sw128_off(r, c & 7), xs + (int64_t)use[k] * D);
            }
            tc::cp_async_arrive_noinc(&full[st]);
        };
        fetch_src(0, ia);
        if (1 < ntiles) fetch_src(1, ib);
        for (int64_t it = 0; it < ntiles; it += 3) {
            tile(it, ia, ic);
            if (it + 1 < ntiles) tile(it + 1, ib, ia);
            if (it + 2 < ntiles) tile(it + 2, ic, ib);
        }
    } else if (warp == S::MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer
        constexpr uint32_t IDESC = tc::idesc_bf16_f32(128, D, false, false);
        const uint32_t bh = tc::smem_u32(b_hi), bl = tc::smem_u32(b_lo);
        int64_t cur = -1;
        uint32_t nbuild = 0;
        const bool leader = tc::elect_one();   // the warp runs the loop; descriptors stay warp-uniform
        for (int64_t it = 0; it < ntiles; ++it) {
            const int st = (int)(it % ST), acc = (int)(it & 1);
            const int64_t ks = kslab_of(first + it);
            if (ks != cur) {
                if (it > 0 && leader) tc::mma_commit(bfree);   // old B free once prior MMAs finish
                tc::mbar_wait(bready, nbuild & 1);
                ++nbuild;
                cur = ks;
            }
            tc::mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
            if (it < 10) stamp(3 + 5 * (int)it);
            if (it >= 2) tc::mbar_wait(&tempty[acc], (uint32_t)(((it >> 1) - 1) & 1));
            tc::fence_proxy_async_smem();          // cp.async (generic proxy) -> tcgen05 (async proxy)
            tc::tc_fence_after();
            {
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * D);
                const uint32_t a = tc::smem_u32(a_base + st * S::TILE_BYTES);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t aoff = (k >> 2) * S::BLK_BYTES + (k & 3) * 32;   // 64-wide K block, 16-elem step
                    const uint32_t boff = (k >> 2) * S::BBLK_BYTES + (k & 3) * 32;
                    const uint64_t da = tc::sw128_desc(a + aoff, 16, 1024);
                    const uint64_t dh = tc::sw128_desc(bh + boff, 16, 1024), dl = tc::sw128_desc(bl + boff, 16, 1024);
                    if (leader) {
                        tc::mma_bf16_ss(d_tmem, da, dh, IDESC, k > 0 ? 1u : 0u);
                        tc::mma_bf16_ss(d_tmem, da, dl, IDESC, 1u);
                    }
                }
                if (leader) {
                    tc::mma_commit(&empty[st]);
                    tc::mma_commit(&tfull[acc]);
                }
                if (it < 10) stamp(4 + 5 * (int)it);
            }
            __syncwarp();
        }
    } else if (warp < 4) {
        // ------------------------------------------------------------------ epilogue (+ B build)
        const int row = tid;                       // TMEM lane = tile row
        int64_t cur = -1;
        uint32_t nbuild = 0;
        for (int64_t it = 0; it < ntiles; ++it) {
            const int64_t id = first + it;
            const int acc = (int)(it & 1);
            const int64_t ks = kslab_of(id);
            if (ks != cur) {
                if (it > 0) tc::mbar_wait(bfree, (nbuild - 1) & 1);
                const int jj = job_of(id);
                const K1TcJob& jb = p.job[jj];
                const int64_t slab = (id - p.job_tile0[jj]) / jb.tiles_per_slab;
                const int H = jb.n_heads, G = H / jb.key_heads;
                const int64_t b = slab / H;
                const uint8_t* sc = scrambler_ptr(jb.keys, jb.keys_bstride, b, (int)((slab % H) / G), D, jb.which);
                // the four tables (s_in, s_out, P1, P2^-1) into SMEM once, then B from SMEM: the
                // 16 K-chunks per thread no longer wait on global loads
                float* const kt_in = reinterpret_cast<float*>(smem + S::OFF_KT);
                float* const kt_out = kt_in + D;
                uint16_t* const kt_p1 = reinterpret_cast<uint16_t*>(kt_out + D);
                uint16_t* const kt_p2 = kt_p1 + D;
                {
                    const float* fin_g = reinterpret_cast<const float*>(sc) + (jb.inv_t ? kInInvT : kInFwd) * D;
                    const float* fout_g = reinterpret_cast<const float*>(sc) + (jb.inv_t ? kOutInvT : kOutFwd) * D;
                    const uint16_t* utab_g = reinterpret_cast<const uint16_t*>(sc + 24 * D);
                    for (int i = tid; i < D; i += 128) {
                        kt_in[i] = fin_g[i];
                        kt_out[i] = fout_g[i];
                        kt_p1[i] = utab_g[kP1 * D + i];
                        kt_p2[i] = utab_g[kP2Inv * D + i];
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                }
                const float* fin = kt_in;
                for (int e = tid; e < D * CPR; e += 128) {
                    const int n = e / CPR, c = e % CPR;   // B row n (output column), K chunk c
                    const uint32_t pn = kt_p2[n];
                    const float on = kt_out[n];
                    uint4 hv, lv;
                    uint32_t* hw = reinterpret_cast<uint32_t*>(&hv);
                    uint32_t* lw = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int i0 = 8 * c + 2 * j, i1 = i0 + 1;
                        const float v0 = ((__popc(kt_p1[i0] & pn) & 1) ? -fin[i0] : fin[i0]) * on;
                        const float v1 = ((__popc(kt_p1[i1] & pn) & 1) ? -fin[i1] : fin[i1]) * on;
                        hw[j] = tc::pack_bf16(v0, v1);
                        float h0, h1;
                        bf16x2_to_f2(hw[j], h0, h1);
                        lw[j] = tc::pack_bf16(v0 - h0, v1 - h1);
                    }
                    const uint32_t off = (c >> 3) * S::BBLK_BYTES + tc::sw128_off(n, c & 7);
                    *reinterpret_cast<uint4*>(b_hi + off) = hv;
                    *reinterpret_cast<uint4*>(b_lo + off) = lv;
                }
                tc::fence_proxy_async_smem();
                tc::mbar_arrive(bready);
                if (warp == 0 && nbuild == 0) stamp(1);
                ++nbuild;
                cur = ks;
            }
            // the output staging is free once the previous tile's TMA store has read it
            if (tid == 0) tc::bulk_wait_read0();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            tc::mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
            tc::tc_fence_after();
            if (warp == 0 && it < 10) stamp(5 + 5 * (int)it);
            uint8_t* o = ostg;
#pragma unroll
            for (int cc = 0; cc < D / 16; ++cc) {
                uint32_t r[16];
                tc::tmem_ld16(tmem_base + (uint32_t)(acc * D + cc * 16) + ((uint32_t)(warp * 32) << 16), r);
                tc::tmem_ld_wait();
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    uint4 w;
                    w.x = tc::pack_bf16(__uint_as_float(r[half * 8 + 0]), __uint_as_float(r[half * 8 + 1]));
                    w.y = tc::pack_bf16(__uint_as_float(r[half * 8 + 2]), __uint_as_float(r[half * 8 + 3]));
                    w.z = tc::pack_bf16(__uint_as_float(r[half * 8 + 4]), __uint_as_float(r[half * 8 + 5]));
                    w.w = tc::pack_bf16(__uint_as_float(r[half * 8 + 6]), __uint_as_float(r[half * 8 + 7]));
                    const int c8 = cc * 2 + half;
                    *reinterpret_cast<uint4*>(o + (c8 >> 3) * S::BLK_BYTES + tc::sw128_off(row, c8 & 7)) = w;
                }
            }
            tc::tc_fence_before();
            tc::mbar_arrive(&tempty[acc]);          // accumulator may be overwritten
            tc::fence_proxy_async_smem();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int jj = job_of(id);
            const K1TcJob& jb = p.job[jj];
            const int64_t lid = id - p.job_tile0[jj];
            const int64_t slab = lid / jb.tiles_per_slab, t = lid % jb.tiles_per_slab;
            const int nrows = tile_rows(jb, lid);
            const int64_t orow0 = slab * jb.out_rows_cap + jb.out_row_offset + t * S::TILE;
            if (nrows == S::TILE) {
                if (tid == 0) {
                    const CUtensorMap* om = &maps.m[jj];
#pragma unroll
                    for (int cb = 0; cb < S::KB; ++cb)
                        tc::tma_store_2d(om, o + cb * S::BLK_BYTES, cb * 64, (int)orow0);
                    tc::bulk_commit();
                    if (it < 10) stamp(6 + 5 * (int)it);
                }
            } else if (tid < nrows) {  // partial tile: never write past the segment
#pragma unroll
                for (int c8 = 0; c8 < CPR; ++c8)
                    *reinterpret_cast<uint4*>(jb.out + (orow0 + tid) * D + c8 * 8) =
                        *reinterpret_cast<const uint4*>(o + (c8 >> 3) * S::BLK_BYTES + tc::sw128_off(tid, c8 & 7));
            }
        }
        if (tid == 0) tc::bulk_wait0();   // this CTA's TMA stores have completed
        if (p.epoch) {
            // remote jobs: make this CTA's stores (TMA and the masked tail) visible system-wide,
            // then count its tiles per job; the CTA completing a job raises the job's flag
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence_system();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (tid == 0) {
                for (int jj = job_of(first); jj < p.n_jobs && p.job_tile0[jj] < last; ++jj) {
                    if (!p.peer_flag[jj]) continue;
                    const int64_t lo = max(first, p.job_tile0[jj]), hi = min(last, p.job_tile0[jj + 1]);
                    const unsigned n = (unsigned)(hi - lo), total = (unsigned)(p.job_tile0[jj + 1] - p.job_tile0[jj]);
                    if (n && atomicAdd(&p.job_counters[jj], n) + n == total) {
                        p.job_counters[jj] = 0;
                        __threadfence_system();
                        flag_raise(p.peer_flag[jj], *p.epoch);
                    }
                }
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

// 2D bf16 tensor map over a row-major [rows x cols] matrix, box {64, box_rows}, 128B swizzle.
bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int num_sms() { return device_sms(); }

template <int D>
static cudaError_t launch_k1_tc_d(const K1Params* qs, const int64_t* n_batch, int n_jobs, cudaStream_t st,
                                  uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* counters) {
    using S = K1TcShape<D>;
    {
        const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k1_tc_kernel<D>), S::SMEM);
        if (e != cudaSuccess) return e;
    }
    if (n_jobs < 1 || n_jobs > kK1Jobs) return cudaErrorInvalidValue;
    K1TcParams p{};
    K1OutMaps maps;
    p.n_jobs = n_jobs;
    p.epoch = epoch;
    p.job_counters = counters;
    int64_t tile0 = 0;
    for (int j = 0; j < kK1Jobs; ++j) {
        p.job_tile0[j] = tile0;
        if (j >= n_jobs) continue;
        const K1Params& q = qs[j];
        K1TcJob& jb = p.job[j];
        jb.x = static_cast<const __nv_bfloat16*>(q.x);
        jb.out = static_cast<__nv_bfloat16*>(q.out);
        jb.keys = static_cast<const uint8_t*>(q.keys);
        jb.perm = q.perm;
        jb.keys_bstride = q.keys_bstride;
        jb.perm_bstride = q.perm_bstride;
        jb.rows = q.rows;
        jb.out_rows_cap = q.out_rows_cap;
        jb.out_row_offset = q.out_row_offset;
        jb.n_heads = q.n_heads;
        jb.key_heads = q.key_heads;
        jb.which = q.which;
        jb.inv_t = q.inv_t;
        jb.x_batch_mod = q.x_batch_mod;
        jb.tiles_per_slab = (q.rows + 127) / 128;
        tile0 += jb.tiles_per_slab * n_batch[j] * q.n_heads;
        if (!make_tmap_bf16_2d(&maps.m[j], q.out, n_batch[j] * q.n_heads * q.out_rows_cap, D, 128))
            return cudaErrorInvalidValue;
        p.peer_flag[j] = peer_flag ? peer_flag[j] : nullptr;
    }
    p.job_tile0[kK1Jobs] = tile0;
    for (int j = n_jobs; j < kK1Jobs; ++j) maps.m[j] = maps.m[0];
    p.total_tiles = tile0;
    p.trace = getenv("SDA_K1TC_TRACE") != nullptr;
    if (p.total_tiles == 0) return cudaSuccess;
    const int64_t grid = std::min<int64_t>(p.total_tiles, num_sms());
    p.tiles_per_cta = (p.total_tiles + grid - 1) / grid;
    const int64_t ngrid = (p.total_tiles + p.tiles_per_cta - 1) / p.tiles_per_cta;
    k1_tc_kernel<D><<<(unsigned)ngrid, S::THREADS, S::SMEM, st>>>(p, maps);
    return cudaGetLastError();
}

bool k1_tc_eligible(const K1Params& p, int d, int xdt, int odt) {
    return xdt == SDA_BF16 && odt == SDA_BF16 && (d == 64 || d == 128) && p.rows >= 128;
}

cudaError_t launch_k1_tc(const K1Params& p, int d, int64_t n_batch, cudaStream_t st) {
    return launch_k1_tc_multi(&p, &n_batch, 1, d, st, nullptr, nullptr, nullptr);
}

cudaError_t launch_k1_tc_multi(const K1Params* p, const int64_t* n_batch, int n_jobs, int d, cudaStream_t st,
                               uint32_t* const* peer_flag, const uint32_t* epoch, uint32_t* counters) {
    if (d == 64) return launch_k1_tc_d<64>(p, n_batch, n_jobs, st, peer_flag, epoch, counters);
    if (d == 128) return launch_k1_tc_d<128>(p, n_batch, n_jobs, st, peer_flag, epoch, counters);
    return cudaErrorInvalidValue;
}

}  // namespace sda

// debug: the last traced K1 launch's per-CTA clock64 stamps (n_cta x 64)
extern "C" int sda_debug_k1tc_trace(unsigned long long* host, int n_cta) {
    if (n_cta > 256) n_cta = 256;
    return cudaMemcpyFromSymbol(host, sda::g_k1tc_trace, sizeof(unsigned long long) * sda::kK1TraceSlots * n_cta) ==
                   cudaSuccess
               ? 0
               : 1;
}
