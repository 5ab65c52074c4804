"""K2 prefill on tcgen05 (k2_prefill_tc.cu): partial attention for many query rows against the
oracle's shard_attention (per split), the SIMT kernel, and the composed scrambled prefill."""
import os

import numpy as np
import pytest
import torch

from oracle import C
from paper_2605_25716_b200 import ops
from tests.gpu_helpers import LSE_TOL, assert_lse, Case, dev, gauss, max_abs_rel, rel_fro

pytestmark = pytest.mark.gpu


def _k2(q, k, v, kv_len, n_splits, simt=False, grouped=False):
    old = os.environ.get("SDA_K2_SIMT")
    if simt:
        os.environ["SDA_K2_SIMT"] = "1"
    else:
        os.environ.pop("SDA_K2_SIMT", None)
    if grouped:
        os.environ["SDA_K2_GROUPED"] = "1"
    else:
        os.environ.pop("SDA_K2_GROUPED", None)
    try:
        o, st = ops.partial_attention(dev(q, torch.bfloat16), dev(k, torch.bfloat16), dev(v, torch.bfloat16),
                                      torch.from_numpy(np.asarray(kv_len, np.int32)).cuda(), n_splits=n_splits)
        torch.cuda.synchronize()
        return o.double().cpu().numpy(), st.double().cpu().numpy()
    finally:
        if old is None:
            os.environ.pop("SDA_K2_SIMT", None)
        else:
            os.environ["SDA_K2_SIMT"] = old


@pytest.mark.parametrize("lq,cap,kv_len,n_splits,hq,hkv", [
    (128, 1024, [1024], 1, 2, 2),
    (300, 1000, [1000, 517], 3, 4, 2),
    (64, 4096, [4096], 2, 2, 1),
    (256, 2048, [129, 2048], 4, 2, 2),
    (513, 384, [384], 1, 1, 1),
])
def test_prefill_tc_vs_oracle(lq, cap, kv_len, n_splits, hq, hkv):
    _check_vs_oracle(lq, cap, kv_len, n_splits, hq, hkv)


@pytest.mark.parametrize("lq,cap,kv_len,n_splits,hq,hkv", [
    (512, 1024, [1024], 2, 2, 2),            # split grid, two 256-row pairs per head = one cluster
    (1024, 4096, [4096, 3000], 1, 4, 4),     # stream-K, groups of 4 CTAs = 2 clusters
    (1024, 2000, [2000, 77], 3, 4, 2),       # split grid, ragged kv_len, GQA
])
def test_prefill_tc_pair_form_vs_oracle(lq, cap, kv_len, n_splits, hq, hkv, monkeypatch):
    """The opt-in CTA-pair form (SDA_K2_PAIR=1: M = 256 tcgen05.mma over a cluster of two CTAs,
    each holding half of every K / V tile, P in shared memory) against the oracle."""
    monkeypatch.setenv("SDA_K2_PAIR", "1")
    _check_vs_oracle(lq, cap, kv_len, n_splits, hq, hkv)


def _check_vs_oracle(lq, cap, kv_len, n_splits, hq, hkv):
    B, d = len(kv_len), 128
    q = C.round_to_format(gauss(31, (B, hq, lq, d)), 2)
    k = C.round_to_format(gauss(32, (B, hkv, cap, d)), 2)
    v = C.round_to_format(gauss(33, (B, hkv, cap, d)), 2)
    o, st = _k2(q, k, v, kv_len, n_splits)
    G = hq // hkv
    for b in range(B):
        L = kv_len[b]
        ntile = -(-L // 128)
        tps = -(-ntile // n_splits)
        for h in range(hq):
            for s in range(n_splits):
                a, e = s * tps * 128, min(L, (s + 1) * tps * 128)
                if a >= e:
                    assert np.all(st[s, b, h, :, 1] == 0)
                    continue
                ro, rm, rs = C.shard_attention(q[b, h], k[b, h // G, a:e], v[b, h // G, a:e])
                # P is rounded to bf16 before the PV product (as every tensor-core flash kernel)
                assert max_abs_rel(o[s, b, h], ro) < 1e-2, (b, h, s)
                assert rel_fro(o[s, b, h], ro) < 5e-3
                assert np.allclose(st[s, b, h, :, 0], rm, atol=1e-3)
                assert_lse(st[s, b, h], rm, rs, LSE_TOL['bf16'], (b, h))


def test_prefill_tc_matches_simt_merged():
    B, H, lq, cap, d = 1, 2, 200, 3000, 128
    q = C.round_to_format(gauss(41, (B, H, lq, d)), 2) * 2
    k = C.round_to_format(gauss(42, (B, H, cap, d)), 2)
    v = C.round_to_format(gauss(43, (B, H, cap, d)), 2)
    a_o, a_s = _k2(q, k, v, [cap], 3)
    b_o, b_s = _k2(q, k, v, [cap], 3, simt=True)
    merged = []
    for o, s in ((a_o, a_s), (b_o, b_s)):
        w = s[..., 1] * np.exp(s[..., 0] - s[..., 0].max(0))
        merged.append((o * w[..., None]).sum(0) / w.sum(0)[..., None])
    assert max_abs_rel(merged[0], merged[1]) < 1e-2 and rel_fro(merged[0], merged[1]) < 5e-3


def test_scrambled_prefill_end_to_end_tc():
    """2 domains x 640-key shards, 300-row prefill span with p_q / p_kv permutations, bf16."""
    case = Case(B=1, Hq=4, Hkv=2, d=128, lk=640, n_nodes=2, lq=300, dtype=torch.bfloat16, seed=21)
    got = case.run_device(n_splits=2)
    ref = case.oracle()
    assert max_abs_rel(got, ref) < 2e-2 and rel_fro(got, ref) < 2e-2


@pytest.mark.parametrize("grouped", [False, True])
@pytest.mark.parametrize("hq,hkv,lq,cap,kv_len,n_splits", [
    (16, 2, 1, 4096, [4096, 1000], 4),     # G=8 decode
    (64, 8, 1, 2048, [2048], 2),           # BASELINE cfg5 head layout
    (8, 1, 4, 1536, [1536], 3),            # G*Lq = 32 (multi-row decode)
    (8, 2, 16, 1024, [700], 2),            # G*Lq = 64
])
def test_gqa_grouped_decode_tc(hq, hkv, lq, cap, kv_len, n_splits, grouped):
    """GQA decode: the swapped kernel (keys on M, k2_gqa_tc.cu; G*Lq <= 32) and the grouped-row
    mode of the prefill kernel (G*Lq <= 128) against the oracle and the SIMT kernel."""
    B, d = len(kv_len), 128
    q = C.round_to_format(gauss(51, (B, hq, lq, d)), 2)
    k = C.round_to_format(gauss(52, (B, hkv, cap, d)), 2)
    v = C.round_to_format(gauss(53, (B, hkv, cap, d)), 2)
    o, st = _k2(q, k, v, kv_len, n_splits, grouped=grouped)
    simt_o, simt_st = _k2(q, k, v, kv_len, n_splits, simt=True)
    G = hq // hkv
    for b in range(B):
        L = kv_len[b]
        ntile = -(-L // 128)
        tps = -(-ntile // n_splits)
        for h in range(hq):
            for s in range(n_splits):
                a, e = s * tps * 128, min(L, (s + 1) * tps * 128)
                if a >= e:
                    assert np.all(st[s, b, h, :, 1] == 0)
                    continue
                ro, rm, rs = C.shard_attention(q[b, h], k[b, h // G, a:e], v[b, h // G, a:e])
                assert max_abs_rel(o[s, b, h], ro) < 1e-2, (b, h, s)
                assert np.allclose(st[s, b, h, :, 0], rm, atol=1e-3)
                assert_lse(st[s, b, h], rm, rs, LSE_TOL['bf16'], (b, h))
    # merged over splits, the grouped tensor-core kernel and the SIMT kernel agree
    def merged(o_, st_):
        m = np.where(st_[..., 1] > 0, st_[..., 0], -np.inf)
        w = st_[..., 1] * np.exp(m - m.max(0))
        return (o_ * w[..., None]).sum(0) / w.sum(0)[..., None]
    a, b_ = merged(o, st), merged(simt_o, simt_st)
    assert max_abs_rel(a, b_) < 1e-2 and rel_fro(a, b_) < 5e-3


def _merge_np(o, st):
    m = np.where(st[..., 1] > 0, st[..., 0], -np.inf)
    mx = m.max(0)
    w = np.where(st[..., 1] > 0, st[..., 1] * np.exp(m - np.where(np.isfinite(mx), mx, 0)), 0.0)
    L = w.sum(0)
    out = (o * w[..., None]).sum(0) / np.where(L > 0, L, 1)[..., None]
    return out, mx, L


@pytest.mark.parametrize("lq,lk,off,n_splits,hq,hkv", [
    (300, 300, 0, 1, 2, 2),       # the inquirer's own span (q_first_pos == k_first_pos)
    (512, 512, 0, 2, 2, 1),       # GQA heads, two splits
    (256, 1000, 744, 1, 1, 1),    # a span at the end of a longer local context
    (200, 200, -5, 3, 2, 2),      # negative offset: the first 5 rows see no key
])
def test_prefill_tc_causal(lq, lk, off, n_splits, hq, hkv):
    """AttentionMask::causal(offset) on the tensor-core prefill kernel (per-row key limits in the
    softmax, tiles past a pair's last visible key skipped) against shard_attention(..., causal)."""
    d = 128
    q = C.round_to_format(gauss(81, (1, hq, lq, d)), 2)
    k = C.round_to_format(gauss(82, (1, hkv, lk, d)), 2)
    v = C.round_to_format(gauss(83, (1, hkv, lk, d)), 2)
    o, st = ops.partial_attention_causal(dev(q, torch.bfloat16), dev(k, torch.bfloat16), dev(v, torch.bfloat16),
                                         causal_offset=off, n_splits=n_splits)
    o, st = o.double().cpu().numpy(), st.double().cpu().numpy()
    mo, mm, ml = _merge_np(o, st)
    G = hq // hkv
    for h in range(hq):
        ro, rm, rs = C.shard_attention(q[0, h], k[0, h // G], v[0, h // G], off)
        live = rs > 0
        assert np.array_equal(ml[0, h] > 0, live), h
        assert max_abs_rel(mo[0, h][live], ro[live]) < 1e-2 and rel_fro(mo[0, h][live], ro[live]) < 5e-3, h
        assert_lse(np.stack([mm[0, h], ml[0, h]], -1), rm, rs, LSE_TOL['bf16'], h)
    # the tensor-core form against the SIMT form of the same call
    os.environ["SDA_K2_SIMT"] = "1"
    try:
        so, sst = ops.partial_attention_causal(dev(q, torch.bfloat16), dev(k, torch.bfloat16), dev(v, torch.bfloat16),
                                               causal_offset=off, n_splits=1)
    finally:
        os.environ.pop("SDA_K2_SIMT", None)
    so = so.double().cpu().numpy()[0]
    live = ml > 0
    assert max_abs_rel(mo[live], so[live]) < 1e-2
