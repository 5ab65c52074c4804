"""K2 prefill in stream-K mode (k2_prefill_tc.cu, one split): persistent CTAs over the units' key
tiles laid end to end, a unit's pieces merged by the last CTA to finish one. Checked against the
oracle's shard_attention over the whole shard, against the split-mode kernel (SDA_K2_NO_SK), for
ragged and empty requests, partial Q tiles, units spread over many CTAs, and repeat launches (the
per-unit tickets reset themselves)."""
import os

import numpy as np
import pytest
import torch

from oracle import C
from paper_2605_25716_b200 import ops
from tests.gpu_helpers import LSE_TOL, assert_lse, dev, gauss, max_abs_rel, rel_fro

pytestmark = pytest.mark.gpu


def _k2(q, k, v, kv_len, sk=True):
    if sk:
        os.environ.pop("SDA_K2_NO_SK", None)
    else:
        os.environ["SDA_K2_NO_SK"] = "1"
    try:
        o, st = ops.partial_attention(dev(q, torch.bfloat16), dev(k, torch.bfloat16), dev(v, torch.bfloat16),
                                      torch.from_numpy(np.asarray(kv_len, np.int32)).cuda(), n_splits=1)
        torch.cuda.synchronize()
        return o[0].double().cpu().numpy(), st[0].double().cpu().numpy()
    finally:
        os.environ.pop("SDA_K2_NO_SK", None)


def _inputs(seed, B, hq, hkv, lq, cap):
    d = 128
    q = C.round_to_format(gauss(seed, (B, hq, lq, d)), 2)
    k = C.round_to_format(gauss(seed + 1, (B, hkv, cap, d)), 2)
    v = C.round_to_format(gauss(seed + 2, (B, hkv, cap, d)), 2)
    return q, k, v


@pytest.mark.parametrize("B,hq,hkv,lq,cap,kv_len", [
    (3, 4, 2, 300, 3000, [1000, 0, 3000]),   # ragged + an empty request; 256 + 44-row Q units
    (1, 8, 8, 512, 4096, [4096]),            # 16 units of 32 tiles over 148 CTAs: ~10 pieces each
    (2, 2, 1, 100, 640, [640, 129]),         # one partial Q tile per unit, tiny ranges
    (1, 1, 1, 64, 128, [1]),                 # a single tile with one key
])
def test_prefill_sk_vs_oracle(B, hq, hkv, lq, cap, kv_len):
    q, k, v = _inputs(61, B, hq, hkv, lq, cap)
    o, st = _k2(q, k, v, kv_len)
    G = hq // hkv
    for b in range(B):
        L = kv_len[b]
        for h in range(hq):
            if L == 0:
                assert np.all(o[b, h] == 0) and np.all(st[b, h, :, 1] == 0) and np.all(np.isneginf(st[b, h, :, 0]))
                continue
            ro, rm, rs = C.shard_attention(q[b, h], k[b, h // G, :L], v[b, h // G, :L])
            assert max_abs_rel(o[b, h], ro) < 1e-2, (b, h)
            assert rel_fro(o[b, h], ro) < 5e-3
            assert np.allclose(st[b, h, :, 0], rm, atol=1e-3)
            assert_lse(st[b, h], rm, rs, LSE_TOL['bf16'], (b, h))


def test_prefill_sk_matches_split_mode_and_repeats():
    """Units spanning one or two CTAs (groups of 8 CTAs over 32 (request, head) x 32 tiles): close to the split-mode
    kernel, and bit-identical across repeated launches (fixed merge order, tickets reset)."""
    q, k, v = _inputs(71, 2, 16, 16, 2048, 4096)
    kv_len = [4096, 3000]
    a_o, a_s = _k2(q, k, v, kv_len)
    b_o, b_s = _k2(q, k, v, kv_len, sk=False)
    # pieces round their own P to bf16 against their own running max: bf16-level differences
    assert max_abs_rel(a_o, b_o) < 1e-2 and rel_fro(a_o, b_o) < 2e-3
    assert np.allclose(a_s[..., 0], b_s[..., 0], atol=1e-5)
    assert np.allclose(a_s[..., 1], b_s[..., 1], rtol=2e-3)
    for _ in range(2):
        c_o, c_s = _k2(q, k, v, kv_len)
        assert np.array_equal(a_o, c_o) and np.array_equal(a_s, c_s)


def test_prefill_sk_whole_units_bit_identical():
    """148 heads x 4 tiles, one Q-tile pair, on 148 SMs: every CTA range is exactly one unit, so
    stream-K copies each unit's result through unchanged -- bit-identical to the split-mode kernel."""
    if torch.cuda.get_device_properties(0).multi_processor_count != 148:
        pytest.skip("needs 148 SMs")
    q, k, v = _inputs(81, 1, 148, 148, 128, 512)
    a_o, a_s = _k2(q, k, v, [512])
    b_o, b_s = _k2(q, k, v, [512], sk=False)
    assert np.array_equal(a_o, b_o) and np.array_equal(a_s, b_s)


def test_prefill_workspace_abi():
    """The C ABI: sda_prefill_workspace_bytes sizes the stream-K workspace (0 for shapes that do not
    run it); sda_partial_attention_ws with it, without it (split grid) and with a too-small one
    (split grid) agree, and the workspace is left zeroed."""
    from paper_2605_25716_b200 import capi
    B, hq, hkv, lq, cap = 1, 4, 4, 512, 2048
    n = int(capi.LIB.sda_prefill_workspace_bytes(B, hq, hkv, lq, cap, 128, capi.SDA_BF16, capi.SDA_BF16))
    assert n > 0
    assert capi.LIB.sda_prefill_workspace_bytes(B, hq, hkv, 1, cap, 128, capi.SDA_BF16, capi.SDA_BF16) == 0
    assert capi.LIB.sda_prefill_workspace_bytes(B, hq, hkv, lq, cap, 64, capi.SDA_BF16, capi.SDA_BF16) == 0
    q, k, v = (dev(x, torch.bfloat16) for x in _inputs(91, B, hq, hkv, lq, cap))
    ws = torch.zeros(n, dtype=torch.uint8, device="cuda")
    outs = []
    for w, nb in ((ws, n), (None, 0), (ws, n - 1)):
        o = torch.empty((1, B, hq, lq, 128), dtype=torch.float32, device="cuda")
        st = torch.empty((1, B, hq, lq, 2), dtype=torch.float32, device="cuda")
        rc = capi.LIB.sda_partial_attention_ws(torch.cuda.current_stream().cuda_stream, q.data_ptr(), capi.SDA_BF16,
                                               k.data_ptr(), v.data_ptr(), capi.SDA_BF16, cap, None, B, hq, hkv, lq,
                                               128, 1, o.data_ptr(), st.data_ptr(),
                                               None if w is None else w.data_ptr(), nb)
        assert rc == 0
        torch.cuda.synchronize()
        outs.append((o.double().cpu().numpy(), st.double().cpu().numpy()))
    # the scratch slots keep the last partials; the leading per-unit tickets must be back at zero
    tick = ws[:4 * (B * hq * ((lq + 255) // 256))].view(torch.int32)
    assert int(tick.abs().sum()) == 0
    for o, st in outs[1:]:
        assert max_abs_rel(outs[0][0], o) < 1e-2 and rel_fro(outs[0][0], o) < 5e-3
        assert np.allclose(outs[0][1][..., 0], st[..., 0], atol=1e-5)


@pytest.mark.parametrize("seed", range(8))
def test_prefill_sk_random_shapes(seed):
    """Seeded random shapes -- ragged and empty requests, GQA, partial Q tiles, units spread over
    one to many CTA groups -- stream-K against the split-grid kernel on the same inputs."""
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 4))
    hkv = int(rng.choice([1, 2, 4]))
    hq = hkv * int(rng.choice([1, 2, 4]))
    lq = int(rng.choice([64, 100, 128, 200, 256, 300, 512, 777]))
    cap = int(rng.choice([128, 640, 1000, 2048, 5000]))
    kv_len = [int(x) for x in rng.integers(0, cap + 1, size=B)]
    kv_len[int(rng.integers(0, B))] = cap
    q, k, v = _inputs(2000 + seed, B, hq, hkv, lq, cap)
    a_o, a_s = _k2(q, k, v, kv_len)
    b_o, b_s = _k2(q, k, v, kv_len, sk=False)
    for b in range(B):
        if kv_len[b] == 0:
            assert np.all(a_o[b] == 0) and np.all(a_s[b, ..., 1] == 0)
            continue
        assert max_abs_rel(a_o[b], b_o[b]) < 1e-2 and rel_fro(a_o[b], b_o[b]) < 5e-3, (b, B, hq, hkv, lq, cap, kv_len)
        assert np.allclose(a_s[b, ..., 0], b_s[b, ..., 0], atol=1e-5)
        assert np.allclose(a_s[b, ..., 1], b_s[b, ..., 1], rtol=5e-3)
