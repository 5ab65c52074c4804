// gpu_scrambled_attn.cpp -- see gpu_scrambled_attn.hpp.
#include "gpu_scrambled_attn.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sdattn_b200.h"

namespace sdattn_b200 {
namespace {

void ck(int st, const char* what) {
    if (st != SDA_OK) throw std::runtime_error(std::string(what) + ": " + sda_status_string(st));
}
void ckc(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer owned by the adapter.
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t bytes) : n(bytes) { ckc(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

std::unique_ptr<DevBuf> upload_f32(const sdattn::Matrix& m) {
    std::vector<float> h(m.data.begin(), m.data.end());
    auto d = std::make_unique<DevBuf>(h.size() * sizeof(float));
    ckc(cudaMemcpy(d->p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    return d;
}

std::unique_ptr<DevBuf> upload_u32(const std::vector<uint32_t>& v) {
    auto d = std::make_unique<DevBuf>(v.size() * 4);
    ckc(cudaMemcpy(d->p, v.data(), v.size() * 4, cudaMemcpyHostToDevice), "H2D");
    return d;
}

// Packed device key image of head `head` for (layer) -- derived with n_heads = head + 1 exactly as
// scrambled_attn renegotiates when more heads arrive (per-head derivation is independent).
struct HeadKeys {
    std::unique_ptr<DevBuf> image;   // SDA_KEYSET_HEAD_BYTES(d): [phi_kq | phi_v] of this head
    uint64_t token_perm_seed = 0;
};

HeadKeys derive_head(const sdattn::ScrambledAttnOptions& opt, size_t layer, size_t head, size_t d) {
    const uint32_t H = static_cast<uint32_t>(head + 1);
    std::vector<double> f(8 * H * d);
    std::vector<uint32_t> u(8 * H * d);
    sda_host_keyset ks{f.data(), u.data(), u.data() + H * d, f.data() + H * d,
                       f.data() + 2 * H * d, u.data() + 2 * H * d, u.data() + 3 * H * d, f.data() + 3 * H * d, 0};
    sda_keyspec spec{1, static_cast<uint32_t>(layer), 0, H, static_cast<uint32_t>(d), opt.mag_lo, opt.mag_hi,
                     opt.scrambler_mode == 1 ? SDA_MODE_S1_ONLY : SDA_MODE_S1_AND_S2};
    ck(sda_negotiate_keyset(opt.shared_seed, &spec, &ks), "negotiate_keyset");
    std::vector<uint8_t> img(sda_keyset_bytes(H, static_cast<uint32_t>(d)));
    ck(sda_pack_keyset(&ks, H, static_cast<uint32_t>(d), img.data()), "pack_keyset");
    HeadKeys hk;
    const size_t hb = SDA_KEYSET_HEAD_BYTES(d);
    hk.image = std::make_unique<DevBuf>(hb);
    ckc(cudaMemcpy(hk.image->p, img.data() + head * hb, hb, cudaMemcpyHostToDevice), "H2D keys");
    hk.token_perm_seed = ks.token_perm_seed;
    return hk;
}

std::vector<uint32_t> span_perm(uint64_t tps, uint64_t tag, uint64_t first, size_t len) {
    std::vector<uint32_t> p(len);
    ck(sda_span_perm(tps, tag, first, len, p.data()), "span_perm");
    return p;
}

}  // namespace

sdattn::AttnFn gpu_scrambled_attn(const sdattn::ScrambledAttnOptions& opt) {
    if (opt.wire_fmt == sdattn::FloatFormat::f16 && opt.quant_bits <= 0)
        throw std::invalid_argument("gpu_scrambled_attn: f16 wire not supported");
    if (opt.quant_bits > 0 && (opt.quant_bits < 2 || opt.quant_bits > 8))
        throw std::invalid_argument("quantize_affine: bits must be in [2, 8]");
    // quantised wire (wire_round, model.cpp:338-341): Q', K', V', O' travel as per-tensor affine
    // codes -> Q', K', V' quantised and dequantised in K1's epilogue (sda_scramble_quant), O' of
    // each shard by a round trip after K2; the normalisation scalars ride at f32
    // (wire_round_stat, model.cpp:343-348)
    const int qbits = opt.quant_bits > 0 ? opt.quant_bits : 0;
    const int dt = (opt.wire_fmt == sdattn::FloatFormat::bf16 && !qbits) ? SDA_BF16 : SDA_F32;
    const size_t esz = dt == SDA_BF16 ? 2 : 4;
    auto keys = std::make_shared<std::map<std::pair<size_t, size_t>, HeadKeys>>();
    return [opt, dt, esz, keys, qbits](const sdattn::AttnRequest& req) -> sdattn::Matrix {
        const size_t d = req.q->cols, lq = req.q->rows, lk = req.k->rows;
        if (d < 4 || d > 256 || (d & (d - 1)))
            throw std::invalid_argument("gpu_scrambled_attn: head dim must be a power of two in [4, 256]");
        auto it = keys->find({req.layer, req.head});
        if (it == keys->end()) it = keys->emplace(std::make_pair(req.layer, req.head), derive_head(opt, req.layer, req.head, d)).first;
        const HeadKeys& hk = it->second;
        cudaStream_t st = nullptr;   // legacy default stream: calls below are ordered

        auto q32 = upload_f32(*req.q);
        const std::vector<uint32_t> pq = span_perm(hk.token_perm_seed, 0, req.q_first_pos, lq);
        std::vector<uint32_t> pq_inv(lq);
        ck(sda_invert_permutation(pq.data(), lq, pq_inv.data()), "invert");
        auto pq_d = upload_u32(pq), pq_inv_d = upload_u32(pq_inv);
        DevBuf q_s(lq * d * esz);
        DevBuf qscratch(16), qerr(4);
        ckc(cudaMemset(qerr.p, 0, 4), "memset");
        // K1; on a quantised wire the quantise -> dequantise of the tensor runs in K1's epilogue
        auto k1 = [&](int variant, int which, const void* x, size_t rows, const uint32_t* perm, void* out, const char* what) {
            if (qbits)
                ck(sda_scramble_quant(st, variant, which, x, SDA_F32, 1, 1, (int64_t)rows, (int)d, hk.image->p, 0, 1, perm,
                                      0, out, dt, (int64_t)rows, 0, 0, qbits, qscratch.as<uint64_t>(), qerr.as<int32_t>()),
                   what);
            else
                ck(sda_scramble(st, variant, which, x, SDA_F32, 1, 1, (int64_t)rows, (int)d, hk.image->p, 0, 1, perm, 0, out,
                                dt, (int64_t)rows, 0, 0),
                   what);
        };
        auto wire = [&](void* x, size_t count) {   // the quantised wire of O', one tensor per shard
            if (qbits)
                ck(sda_quant_roundtrip(st, x, SDA_F32, 1, (int64_t)count, qbits, qscratch.as<uint64_t>(),
                                       qerr.as<int32_t>()),
                   "quant roundtrip");
        };
        k1(SDA_PHI_FORWARD, SDA_KEYS_KQ, q32->p, lq, pq_d->as<uint32_t>(), q_s.p, "scramble Q");

        std::vector<std::unique_ptr<DevBuf>> keep;
        std::vector<sda_merge_source> src;
        for (const sdattn::KVCacheSegment* seg : req.prior) {   // each segment = one remote shard
            const sdattn::Matrix& k = seg->k[req.layer][req.head];
            const sdattn::Matrix& v = seg->v[req.layer][req.head];
            const size_t L = k.rows;
            auto k32 = upload_f32(k), v32 = upload_f32(v);
            auto pkv = upload_u32(span_perm(hk.token_perm_seed, 1, seg->first_pos, L));
            auto ks = std::make_unique<DevBuf>(L * d * esz), vs = std::make_unique<DevBuf>(L * d * esz);
            k1(SDA_PHI_INV_T, SDA_KEYS_KQ, k32->p, L, pkv->as<uint32_t>(), ks->p, "scramble K");
            k1(SDA_PHI_FORWARD, SDA_KEYS_V, v32->p, L, pkv->as<uint32_t>(), vs->p, "scramble V");
            auto o = std::make_unique<DevBuf>(lq * d * 4), s = std::make_unique<DevBuf>(lq * 2 * 4);
            ck(sda_partial_attention(st, q_s.p, dt, ks->p, vs->p, dt, (int64_t)L, nullptr, 1, 1, 1, (int64_t)lq, (int)d, 1,
                                     o->as<float>(), s->as<float>()),
               "partial attention");
            wire(o->p, lq * d);   // O' of the shard (one split)
            if (dt == SDA_BF16) {    // wire_round of O' and wire_round_stat of the stats (model.cpp:392-394)
                ck(sda_wire_round(st, o->p, SDA_F32, (int64_t)(lq * d), 2), "wire_round O'");
                ck(sda_wire_round(st, s->p, SDA_F32, (int64_t)(lq * 2), 2), "wire_round stats");
            }
            src.push_back({o->as<float>(), s->as<float>(), hk.image->p, pq_inv_d->as<uint32_t>(), 0});
            keep.push_back(std::move(ks));
            keep.push_back(std::move(vs));
            keep.push_back(std::move(o));
            keep.push_back(std::move(s));
            keep.push_back(std::move(k32));
            keep.push_back(std::move(v32));
            keep.push_back(std::move(pkv));
        }
        // the inquirer's own span, plaintext (protocol.cpp:944-947; model.cpp:397-398)
        auto k32 = upload_f32(*req.k), v32 = upload_f32(*req.v);
        DevBuf lo(lq * d * 4), ls(lq * 2 * 4);
        if (req.causal)
            ck(sda_partial_attention_causal(st, q32->p, SDA_F32, k32->p, v32->p, SDA_F32, (int64_t)lk, nullptr, 1, 1, 1,
                                            (int64_t)lq, (int)d, 1, 0, lo.as<float>(), ls.as<float>()),
               "local causal shard");
        else
            ck(sda_partial_attention(st, q32->p, SDA_F32, k32->p, v32->p, SDA_F32, (int64_t)lk, nullptr, 1, 1, 1,
                                     (int64_t)lq, (int)d, 1, lo.as<float>(), ls.as<float>()),
               "local shard");
        src.push_back({lo.as<float>(), ls.as<float>(), nullptr, nullptr, 0});

        DevBuf out(lq * d * 4), err(4);
        ckc(cudaMemset(err.p, 0, 4), "memset");
        ck(sda_unscramble_merge(st, src.data(), (int)src.size(), 0, 1, 0, 1, 1, (int64_t)lq, (int)d, out.p, SDA_F32,
                                nullptr, err.as<int32_t>(), 0),
           "unscramble_merge");
        std::vector<float> h(lq * d);
        int32_t e = 0;
        ckc(cudaMemcpy(h.data(), out.p, h.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        ckc(cudaMemcpy(&e, err.p, 4, cudaMemcpyDeviceToHost), "D2H");
        if (e == SDA_ERR_MASKED_ROW) throw std::invalid_argument("merge_shards: row masked in every shard");
        ckc(cudaMemcpy(&e, qerr.p, 4, cudaMemcpyDeviceToHost), "D2H");
        if (e != 0) throw std::invalid_argument("quantize_affine: non-finite value");
        return sdattn::Matrix(lq, d, std::vector<double>(h.begin(), h.end()));
    };
}

}  // namespace sdattn_b200
