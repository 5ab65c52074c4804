"""Out-of-bounds write guards (compute-sanitizer is closed on this GPU pool, so the kernels' own
bounds are checked directly): every output of every kernel family is placed inside a larger
buffer whose guard regions before and after hold a known bit pattern, and the inputs are
fingerprinted; after the launch the guards and the inputs must be bit-identical. Shapes are the
edge cases of each kernel: ragged kv_len and empty splits, partial 128-row tiles and 256-row
pairs, one-row spans, the small head dims, GQA groups, causal tails, the stream-K scratch, the
quantised wire's two passes, the FP64 mode."""
import pytest
import torch

from paper_2605_25716_b200 import capi, ops, protocol

pytestmark = pytest.mark.gpu
G = 8192   # guard elements on each side


class Guarded:
    def __init__(self, shape, dtype):
        n = 1
        for s in shape:
            n *= s
        self.buf = torch.empty(n + 2 * G, dtype=dtype, device="cuda")
        self.buf.view(torch.uint8).fill_(0xA5)
        self.t = self.buf[G:G + n].view(shape)
        self.before = self.buf[:G].clone()
        self.after = self.buf[G + n:].clone()

    def check(self, what):
        torch.cuda.synchronize()
        assert torch.equal(self.buf[:G].view(torch.uint8), self.before.view(torch.uint8)), f"{what}: write before the output"
        assert torch.equal(self.buf[-G:].view(torch.uint8), self.after.view(torch.uint8)), f"{what}: write past the output"


def _fp(*ts):
    return [t.clone() for t in ts]


def _same(a, b, what):
    for x, y in zip(a, b):
        assert torch.equal(x.view(torch.uint8) if x.dtype != torch.bool else x, y.view(torch.uint8) if y.dtype != torch.bool else y), \
            f"{what}: an input was written"


def _rn(g, *s, dt=torch.bfloat16):
    return torch.randn(s, generator=g, device="cuda").to(dt)


@pytest.mark.parametrize("d,dt,rows", [(128, torch.bfloat16, 300), (128, torch.bfloat16, 1), (64, torch.bfloat16, 129),
                                       (16, torch.float32, 45), (4, torch.bfloat16, 7), (32, torch.float32, 1)])
def test_k1_guards(d, dt, rows):
    g = torch.Generator(device="cuda").manual_seed(d + rows)
    keys = protocol.DomainKeys([1, 2, 3], 0, 1, 2, d, "cuda")
    x = _rn(g, 3, 2, rows, d, dt=dt)
    perm, _ = keys.span_perms(1, 5, rows)
    ins = _fp(x, keys.dev, perm)
    out = Guarded((3, 2, rows, d), dt)
    ops.scramble(x, keys.dev, capi.PHI_INV_T, capi.KEYS_KQ, perm, out=out.t)
    out.check("K1")
    _same([x, keys.dev, perm], ins, "K1")
    if dt == torch.float32:
        outq = Guarded((3, 2, rows, d), torch.float32)
        ops.scramble_quant(x, keys.dev, capi.PHI_FORWARD, capi.KEYS_V, 4, perm, out=outq.t)
        outq.check("K1 quant")


@pytest.mark.parametrize("case", ["decode", "decode_small_d", "prefill_split", "prefill_sk", "gqa", "causal_tc",
                                  "causal_simt", "fp64"])
def test_k2_guards(case):
    g = torch.Generator(device="cuda").manual_seed(7)
    d, dt, B, Hq, Hkv, lq, cap, S = 128, torch.bfloat16, 3, 4, 4, 1, 700, 5
    kv_len = torch.tensor([700, 333, 1], dtype=torch.int32, device="cuda")
    if case == "decode_small_d":
        d, dt = 8, torch.float32
    elif case == "prefill_split":
        lq, S = 300, 3
    elif case == "prefill_sk":
        lq, S = 300, 1
    elif case == "gqa":
        Hq, Hkv, S = 16, 2, 3
    elif case.startswith("causal"):
        lq, cap, S, B = 300, 300, 1 if case == "causal_tc" else 2, 1
        kv_len = None
    elif case == "fp64":
        d, dt, lq = 16, torch.float64, 3
    q = _rn(g, B, Hq, lq, d, dt=dt)
    k, v = _rn(g, B, Hkv, cap, d, dt=dt), _rn(g, B, Hkv, cap, d, dt=dt)
    ins = _fp(q, k, v)
    pdt = torch.float64 if dt == torch.float64 else torch.float32
    o = Guarded((S, B, Hq, lq, d), pdt)
    st = Guarded((S, B, Hq, lq, 2), pdt)
    if case.startswith("causal"):
        if case == "causal_simt":
            import os
            os.environ["SDA_K2_SIMT"] = "1"
        try:
            ops.partial_attention_causal(q, k, v, causal_offset=-3, n_splits=S, out_o=o.t, out_stats=st.t)
        finally:
            import os
            os.environ.pop("SDA_K2_SIMT", None)
    else:
        ops.partial_attention(q, k, v, kv_len[:B] if kv_len is not None else None, n_splits=S, out_o=o.t, out_stats=st.t)
    o.check(f"K2 {case} O'")
    st.check(f"K2 {case} stats")
    _same([q, k, v], ins, f"K2 {case}")
    assert torch.isfinite(o.t).all()


@pytest.mark.parametrize("case", ["decode", "rows", "rows_multi", "tiny", "quant_rows", "fp64", "packed", "tc", "tc_d64"])
def test_k3_guards(case, monkeypatch):
    g = torch.Generator(device="cuda").manual_seed(11)
    B, H, lq, d, S = 2, 3, 1, 128, 4
    dt = torch.float32
    if case.startswith("rows") or case == "quant_rows":
        lq = 130
    if case.startswith("tc"):   # the tensor-core form: 2 splits + the plaintext source, a ragged last tile
        monkeypatch.setenv("SDA_K3_TC", "1")
        lq, S = 300, 3
        if case == "tc_d64":
            d = 64
    if case == "rows_multi":
        S = 6
    if case == "tiny":
        d, lq = 8, 5
    if case == "fp64":
        d, lq, dt, S = 16, 4, torch.float64, 2
    keys = [protocol.DomainKeys([1, 2], 0, dom + 1, H, d, "cuda", fp64=dt == torch.float64) for dom in range(2)]
    pinv = None
    if lq > 1:
        _, pinv = keys[0].span_perms(0, 9, lq)
    srcs, ins = [], []
    for s in range(S):
        o = torch.randn((B, H, lq, d), generator=g, device="cuda").to(dt)
        st = torch.stack([torch.randn((B, H, lq), generator=g, device="cuda"),
                          torch.rand((B, H, lq), generator=g, device="cuda") + 0.1], -1).to(dt).contiguous()
        srcs.append(ops.MergeSource(o, st, keys[s % 2 if case == "rows_multi" else 0].dev if s < S - 1 else None,
                                    pinv if s < S - 1 else None))
        ins += [o, st]
    if case == "rows_multi":
        srcs.sort(key=lambda m: -1 if m.keys is None else m.keys.data_ptr())
    saved = _fp(*ins)
    out = Guarded((B, H, lq, d), dt if case == "fp64" else torch.bfloat16)
    ost = Guarded((B, H, lq, 2), dt)
    if case == "packed":   # O' and stats in one packed record per request (the exchange layout)
        # 3 heads x 1 row x 130 floats: the second request's record would start 8 bytes off the
        # 16-byte vector alignment of K3's row loads / stores -- refused, not written misaligned
        rec = Guarded((B, H * lq * (d + 2)), torch.float32)
        with pytest.raises(capi.SdaError):
            ops.unscramble_merge(srcs, out=rec.t, out_stats=rec.t[:, H * lq * d:], out_batch_stride=H * lq * (d + 2),
                                 key_heads=H)
        rec.check("K3 packed (refused)")
        H2 = 4
        srcs = [ops.MergeSource(torch.cat([m.o, m.o[:, :1]], 1).contiguous(), torch.cat([m.stats, m.stats[:, :1]], 1).contiguous(),
                                None if m.keys is None else protocol.DomainKeys([1, 2], 0, 1, H2, d, "cuda").dev,
                                m.pq_inv) for m in srcs]
        ins = [t for m in srcs for t in (m.o, m.stats)]
        saved = _fp(*ins)
        H = H2
        rec = Guarded((B, H * lq * (d + 2)), torch.float32)
        ops.unscramble_merge(srcs, out=rec.t, out_stats=rec.t[:, H * lq * d:], out_batch_stride=H * lq * (d + 2),
                             key_heads=H)
        rec.check("K3 packed")
    else:
        ops.unscramble_merge(srcs, out=out.t, out_stats=ost.t, quant_bits=8 if case == "quant_rows" else 0, key_heads=H)
        out.check(f"K3 {case}")
        ost.check(f"K3 {case} stats")
    _same(ins, saved, f"K3 {case}")
