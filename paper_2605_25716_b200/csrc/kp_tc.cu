// kp_tc.cu -- the QKV projection with K1 fused into it: one tcgen05 kernel computes
//   out[b][h][off + r][:] = bf16( (x[b][perm_b[r]][:] @ W_h^T) phi_{b,h} )
// replacing project_qkv (model.cpp:124-133) followed by enc_qkv's scramble and row gather
// (scrambler.cpp:126-136): the inquirer's span Q (protocol.cpp:885-891) and the context owner's
// K / V shipping (protocol.cpp:993-1001) straight from the layer input, with no unscrambled
// Q / K / V ever written to HBM.
//
// Per CTA = one 128-row tile of one (request, head), 9 warps:
//   warps 4-7 (loaders)  : the prologue's row gather -- cp.async 16-byte chunks of the input rows
//                          x[b][perm_b[r]] into SWIZZLE_128B K-major A stages; lane 0 of warp 4 also
//                          TMA-loads the matching [d x 64] block of W_h (the nn.Linear weight rows
//                          h*d .. h*d+d-1, K-major as stored);
//   warp 8     (MMA)     : Y = A W_h^T over d_model in 64-wide steps (tcgen05.mma, M=128, N=d, K=16)
//                          into TMEM; then the scramble GEMM Z = Y B (below) into a second
//                          TMEM accumulator;
//   warps 0-3  (epilogue): build B for the (request, head)'s key set while the projection runs --
//                          B[n][i] = (-1)^popc(P1[i] & P2inv[n]) s1^{+-1}[i] s2^{+-1}[n] / sqrt(d), split
//                          into bf16 hi + lo as in K1 (k1_tc.cu) -- then Y (f32, TMEM) -> bf16
//                          hi + lo into SMEM, and after the scramble GEMM Z -> bf16 -> TMA store.
// The scramble GEMM runs Y_hi B_hi + Y_hi B_lo + Y_lo B_hi in f32 (~2^-16 relative), so the one
// rounding is the final bf16 store, as in K1.
#include "common.cuh"
#include "tc_util.cuh"

#include <algorithm>

namespace sda {

bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);

struct KpParams {
    const __nv_bfloat16* x;    // [n_batch][x_rows][d_model]
    __nv_bfloat16* out;        // [n_batch][n_heads][out_rows_cap][d]
    const uint8_t* keys;       // request b's key set at keys + b * keys_bstride
    const uint32_t* perm;      // request b's row gather at perm + b * perm_bstride (null: identity)
    int64_t keys_bstride, perm_bstride;
    int64_t rows, x_rows, out_rows_cap, out_row_offset;
    int n_heads, key_heads, which, inv_t, d_model;
};

template <int D>
struct KpShape {
    static constexpr int TILE = 128;
    // projection K stages: a stage is only 4 MMAs (256 tensor cycles) of work, so the loads need
    // many stages in flight to cover their latency (3 stages: 39 % tensor-pipe active, ncu)
    static constexpr int ST = D == 128 ? 5 : 8;
    static constexpr int A_BYTES = TILE * 128;                // [128 x 64] bf16, one K step of A
    static constexpr int B_BYTES = D * 128;                   // [d x 64] bf16, one K step of W_h
    static constexpr int OFF_STAGE = 0;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    // Y hi / lo [128 x d] (K-major, d/64 blocks) reuse the stages: they are written after the last
    // projection MMA has completed (yfull), when no stage is read or loaded any more
    static constexpr int OFF_A2H = 0;
    static constexpr int OFF_A2L = OFF_A2H + TILE * D * 2;
    static_assert(2 * TILE * D * 2 <= ST * STAGE_BYTES, "Y hi / lo must fit in the stages");
    static constexpr int OFF_BH = ST * STAGE_BYTES;           // B hi [d x d]
    static constexpr int OFF_BL = OFF_BH + D * D * 2;
    static constexpr int OFF_KT = OFF_BL + D * D * 2;         // key tables
    static constexpr int OFF_BAR = OFF_KT + D * 12;
    // full[ST], empty[ST], yfull, a2ready, bready, zfull
    static constexpr int NBAR = 2 * ST + 4;
    static constexpr int SMEM = OFF_BAR + 8 * NBAR + 16;
    static constexpr uint32_t TMEM_COLS = 2 * D;
    static constexpr int THREADS = 288;
    static_assert(SMEM <= 232448, "shared memory");
};

template <int D>
__global__ void __launch_bounds__(288, 1) kp_tc_kernel(const KpParams p, const __grid_constant__ CUtensorMap wmap,
                                                       const __grid_constant__ CUtensorMap omap) {
    using S = KpShape<D>;
    constexpr int ST = S::ST, TILE = S::TILE;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* const full = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
    uint64_t* const empty = full + ST;
    uint64_t* const yfull = empty + ST;
    uint64_t* const a2ready = yfull + 1;
    uint64_t* const bready = a2ready + 1;
    uint64_t* const zfull = bready + 1;
    uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(zfull + 1);
    uint8_t* const a2h = smem + S::OFF_A2H;
    uint8_t* const a2l = smem + S::OFF_A2L;
    uint8_t* const bh = smem + S::OFF_BH;
    uint8_t* const bl = smem + S::OFF_BL;

    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    const int h = blockIdx.y;
    const int64_t b = blockIdx.z;
    const int nrows = (int)min((int64_t)TILE, p.rows - tile * TILE);
    const int nk = p.d_model / 64;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            tc::mbar_init(&full[s], 128 + 1);   // the loaders' cp.async arrivals + the W TMA
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(yfull, 1);
        tc::mbar_init(a2ready, 128);
        tc::mbar_init(bready, 128);
        tc::mbar_init(zfull, 1);
        tc::fence_mbar_init();
        tc::prefetch_tmap(&wmap);
        tc::prefetch_tmap(&omap);
    }
    if (warp == 0) tc::tmem_alloc<S::TMEM_COLS>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t COL_Y = 0, COL_Z = D;

    if (warp >= 4 && warp < 8) {
        // ------------------------------------------------------------------ loaders
        const int lt = tid - 128;
        constexpr int CPR = 8;                  // 16-byte chunks per 64-wide row slice
        constexpr int RSTEP = 128 / CPR, NR = TILE / RSTEP;
        const int c = lt % CPR, r0 = lt / CPR;
        int32_t src[NR];
        const uint32_t* pm = p.perm ? p.perm + b * p.perm_bstride + tile * TILE : nullptr;
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int r = r0 + k * RSTEP;
            src[k] = r < nrows ? (pm ? (int32_t)__ldg(pm + r) : (int32_t)(tile * TILE + r)) : -1;
        }
        const __nv_bfloat16* xs = p.x + (b * p.x_rows) * p.d_model + c * 8;
        for (int kk = 0; kk < nk; ++kk) {
            const int st = kk % ST;
            if (kk >= ST) tc::mbar_wait(&empty[st], (uint32_t)(((kk / ST) - 1) & 1));
            uint8_t* a = smem + S::OFF_STAGE + st * S::STAGE_BYTES;
            if (lt == 0) {   // W_h rows h*d .. h*d+d-1, K columns kk*64 .. +63
                tc::mbar_arrive_expect_tx(&full[st], S::B_BYTES);
                tc::tma_load_2d(a + S::A_BYTES, &wmap, kk * 64, h * D, &full[st]);
            }
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const int r = r0 + k * RSTEP;
                if (src[k] >= 0) tc::cp_async16(a + tc::sw128_off(r, c), xs + (int64_t)src[k] * p.d_model + kk * 64);
            }
            tc::cp_async_arrive_noinc(&full[st]);
        }
    } else if (warp == 8) {
        // ------------------------------------------------------------------ MMA issuer
        const bool leader = tc::elect_one();
        constexpr uint32_t IDESC = tc::idesc_bf16_f32(128, D, false, false);
        for (int kk = 0; kk < nk; ++kk) {
            const int st = kk % ST;
            tc::mbar_wait(&full[st], (uint32_t)((kk / ST) & 1));
            tc::fence_proxy_async_smem();   // cp.async (generic proxy) -> tcgen05 (async proxy)
            tc::tc_fence_after();
            const uint32_t a = tc::smem_u32(smem + S::OFF_STAGE + st * S::STAGE_BYTES);
            const uint32_t w = a + S::A_BYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint64_t da = tc::sw128_desc(a + k * 32, 16, 1024), db = tc::sw128_desc(w + k * 32, 16, 1024);
                if (leader) tc::mma_bf16_ss(tmem + COL_Y, da, db, IDESC, (kk > 0 || k > 0) ? 1u : 0u);
            }
            if (leader) tc::mma_commit(&empty[st]);
            __syncwarp();
        }
        if (leader) tc::mma_commit(yfull);
        // the scramble GEMM: Z = Y_hi B_hi + Y_hi B_lo + Y_lo B_hi
        tc::mbar_wait(bready, 0);
        tc::mbar_wait(a2ready, 0);
        tc::tc_fence_after();
        const uint32_t ah = tc::smem_u32(a2h), al = tc::smem_u32(a2l), bhs = tc::smem_u32(bh), bls = tc::smem_u32(bl);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
            const uint32_t aoff = (k >> 2) * (TILE * 128) + (k & 3) * 32;
            const uint32_t boff = (k >> 2) * (D * 128) + (k & 3) * 32;
            const uint64_t dah = tc::sw128_desc(ah + aoff, 16, 1024), dal = tc::sw128_desc(al + aoff, 16, 1024);
            const uint64_t dbh = tc::sw128_desc(bhs + boff, 16, 1024), dbl = tc::sw128_desc(bls + boff, 16, 1024);
            if (leader) {
                tc::mma_bf16_ss(tmem + COL_Z, dah, dbh, IDESC, k > 0 ? 1u : 0u);
                tc::mma_bf16_ss(tmem + COL_Z, dah, dbl, IDESC, 1u);
                tc::mma_bf16_ss(tmem + COL_Z, dal, dbh, IDESC, 1u);
            }
        }
        if (leader) tc::mma_commit(zfull);
        __syncwarp();
    } else if (warp < 4) {
        // ------------------------------------------------------------------ B build, epilogues
        const int row = tid;
        {   // B for (request b, key head of h), as k1_tc.cu builds it
            const int G = p.n_heads / p.key_heads;
            const uint8_t* sc = scrambler_ptr(p.keys, p.keys_bstride, b, h / G, D, p.which);
            float* const kt_in = reinterpret_cast<float*>(smem + S::OFF_KT);
            float* const kt_out = kt_in + D;
            uint16_t* const kt_p1 = reinterpret_cast<uint16_t*>(kt_out + D);
            uint16_t* const kt_p2 = kt_p1 + D;
            const float* fin_g = reinterpret_cast<const float*>(sc) + (p.inv_t ? kInInvT : kInFwd) * D;
            const float* fout_g = reinterpret_cast<const float*>(sc) + (p.inv_t ? kOutInvT : kOutFwd) * D;
            const uint16_t* utab_g = reinterpret_cast<const uint16_t*>(sc + 24 * D);
            for (int i = tid; i < D; i += 128) {
                kt_in[i] = fin_g[i];
                kt_out[i] = fout_g[i];
                kt_p1[i] = utab_g[kP1 * D + i];
                kt_p2[i] = utab_g[kP2Inv * D + i];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            constexpr int CPRB = D / 8;
            for (int e = tid; e < D * CPRB; e += 128) {
                const int n = e / CPRB, c = e % CPRB;
                const uint32_t pn = kt_p2[n];
                const float on = kt_out[n];
                uint4 hv, lv;
                uint32_t* hw = reinterpret_cast<uint32_t*>(&hv);
                uint32_t* lw = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int i0 = 8 * c + 2 * j, i1 = i0 + 1;
                    const float v0 = ((__popc(kt_p1[i0] & pn) & 1) ? -kt_in[i0] : kt_in[i0]) * on;
                    const float v1 = ((__popc(kt_p1[i1] & pn) & 1) ? -kt_in[i1] : kt_in[i1]) * on;
                    hw[j] = tc::pack_bf16(v0, v1);
                    float h0, h1;
                    bf16x2_to_f2(hw[j], h0, h1);
                    lw[j] = tc::pack_bf16(v0 - h0, v1 - h1);
                }
                const uint32_t off = (c >> 3) * (D * 128) + tc::sw128_off(n, c & 7);
                *reinterpret_cast<uint4*>(bh + off) = hv;
                *reinterpret_cast<uint4*>(bl + off) = lv;
            }
            tc::fence_proxy_async_smem();
            tc::mbar_arrive(bready);
        }
        // Y (f32) -> bf16 hi + lo, K-major SW128 A operands of the scramble GEMM
        tc::mbar_wait(yfull, 0);
        tc::tc_fence_after();
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
#pragma unroll
        for (int cc = 0; cc < D / 16; ++cc) {
            uint32_t r[16];
            tc::tmem_ld16(tmem + COL_Y + cc * 16 + lane_off, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint4 hv, lv;
                uint32_t* hw = reinterpret_cast<uint32_t*>(&hv);
                uint32_t* lw = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float v0 = __uint_as_float(r[half * 8 + 2 * j]), v1 = __uint_as_float(r[half * 8 + 2 * j + 1]);
                    hw[j] = tc::pack_bf16(v0, v1);
                    float h0, h1;
                    bf16x2_to_f2(hw[j], h0, h1);
                    lw[j] = tc::pack_bf16(v0 - h0, v1 - h1);
                }
                const int c8 = cc * 2 + half;
                const uint32_t off = (c8 >> 3) * (TILE * 128) + tc::sw128_off(row, c8 & 7);
                *reinterpret_cast<uint4*>(a2h + off) = hv;
                *reinterpret_cast<uint4*>(a2l + off) = lv;
            }
        }
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        tc::mbar_arrive(a2ready);
        // Z -> bf16 -> staging (the Y hi region: the scramble GEMM has read it once zfull fires)
        tc::mbar_wait(zfull, 0);
        tc::tc_fence_after();
        uint8_t* const o = a2h;
#pragma unroll
        for (int cc = 0; cc < D / 16; ++cc) {
            uint32_t r[16];
            tc::tmem_ld16(tmem + COL_Z + cc * 16 + lane_off, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint4 w;
                w.x = tc::pack_bf16(__uint_as_float(r[half * 8 + 0]), __uint_as_float(r[half * 8 + 1]));
                w.y = tc::pack_bf16(__uint_as_float(r[half * 8 + 2]), __uint_as_float(r[half * 8 + 3]));
                w.z = tc::pack_bf16(__uint_as_float(r[half * 8 + 4]), __uint_as_float(r[half * 8 + 5]));
                w.w = tc::pack_bf16(__uint_as_float(r[half * 8 + 6]), __uint_as_float(r[half * 8 + 7]));
                const int c8 = cc * 2 + half;
                *reinterpret_cast<uint4*>(o + (c8 >> 3) * (TILE * 128) + tc::sw128_off(row, c8 & 7)) = w;
            }
        }
        tc::fence_proxy_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int64_t orow0 = (b * p.n_heads + h) * p.out_rows_cap + p.out_row_offset + tile * TILE;
        if (nrows == TILE) {
            if (tid == 0) {
#pragma unroll
                for (int cb = 0; cb < D / 64; ++cb) tc::tma_store_2d(&omap, o + cb * (TILE * 128), cb * 64, (int)orow0);
                tc::bulk_commit();
                tc::bulk_wait0();
            }
        } else if (tid < nrows) {   // partial tile: never write past the span
#pragma unroll
            for (int c8 = 0; c8 < D / 8; ++c8)
                *reinterpret_cast<uint4*>(p.out + (orow0 + tid) * D + c8 * 8) =
                    *reinterpret_cast<const uint4*>(o + (c8 >> 3) * (TILE * 128) + tc::sw128_off(tid, c8 & 7));
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == 0) tc::tmem_dealloc<S::TMEM_COLS>(tmem);
}

template <int D>
static cudaError_t launch_kp_d(const KpParams& p, int64_t n_batch, const void* w, cudaStream_t st) {
    using S = KpShape<D>;
    {
        const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kp_tc_kernel<D>), S::SMEM);
        if (e != cudaSuccess) return e;
    }
    CUtensorMap wm, om;
    if (!make_tmap_bf16_2d(&wm, w, (int64_t)p.n_heads * D, p.d_model, D) ||
        !make_tmap_bf16_2d(&om, p.out, n_batch * p.n_heads * p.out_rows_cap, D, 128))
        return cudaErrorInvalidValue;
    const dim3 grid((unsigned)((p.rows + 127) / 128), (unsigned)p.n_heads, (unsigned)n_batch);
    kp_tc_kernel<D><<<grid, S::THREADS, S::SMEM, st>>>(p, wm, om);
    return cudaGetLastError();
}

cudaError_t launch_project_scramble(const void* x, int64_t n_batch, int64_t x_rows, int d_model, const void* w,
                                    int n_heads, int d, const void* keys, int64_t keys_bstride, int key_heads,
                                    int variant, int which, const uint32_t* perm, int64_t perm_bstride, int64_t rows,
                                    void* out, int64_t out_rows_cap, int64_t out_row_offset, cudaStream_t st) {
    KpParams p{};
    p.x = static_cast<const __nv_bfloat16*>(x);
    p.out = static_cast<__nv_bfloat16*>(out);
    p.keys = static_cast<const uint8_t*>(keys);
    p.perm = perm;
    p.keys_bstride = keys_bstride;
    p.perm_bstride = perm_bstride;
    p.rows = rows;
    p.x_rows = x_rows;
    p.out_rows_cap = out_rows_cap;
    p.out_row_offset = out_row_offset;
    p.n_heads = n_heads;
    p.key_heads = key_heads;
    p.which = which;
    p.inv_t = variant == SDA_PHI_INV_T ? 1 : 0;
    p.d_model = d_model;
    if (d == 128) return launch_kp_d<128>(p, n_batch, w, st);
    if (d == 64) return launch_kp_d<64>(p, n_batch, w, st);
    return cudaErrorInvalidValue;
}

}  // namespace sda
