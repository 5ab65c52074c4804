"""Small head dims (d = 4, 8, 16): the reference's own model / protocol tests run at head_dim 16
(test_model.cpp:17-19, helpers.hpp:19) and its finiteness sweep at 4 / 8 / 16 (test_model.cpp:188).
K1 (SIMT, one lane per row), K2 (SIMT decode form, one lane per key row at d = 4) and K3 (one
thread per row) against the oracle, per kernel and composed."""
import numpy as np
import pytest
import torch

from oracle import C
from paper_2605_25716_b200 import capi, ops
from tests.gpu_helpers import Case, dev, gauss, max_abs_rel, rel_fro

pytestmark = pytest.mark.gpu
DS = [4, 8, 16]


def _keys(B, H, d, domain=1):
    kh = [capi.negotiate_keyset(capi.shared_seed(1, b + 1), b + 1, 0, domain, H, d) for b in range(B)]
    return kh, ops.upload_keys([k.pack() for k in kh], "cuda")


def _sc(ks, h, which):
    p = "kq" if which == 0 else "v"
    return (getattr(ks, p + "_s1")[h], getattr(ks, p + "_p1")[h], getattr(ks, p + "_p2")[h], getattr(ks, p + "_s2")[h])


@pytest.mark.parametrize("d", DS)
@pytest.mark.parametrize("rows", [1, 45])
@pytest.mark.parametrize("variant,which", [(capi.PHI_FORWARD, capi.KEYS_KQ), (capi.PHI_INV_T, capi.KEYS_KQ),
                                           (capi.PHI_FORWARD, capi.KEYS_V)])
def test_k1_small_d_f32(d, rows, variant, which):
    B, H = 3, 2
    kh, kd = _keys(B, H, d)
    x = gauss(3, (B, H, rows, d))
    perms = [kh[b].span_perm(1, 7 * b, rows) for b in range(B)]
    out = ops.scramble(dev(x, torch.float32), kd, variant, which, ops.upload_perms(perms, "cuda"))
    got = out.double().cpu().numpy()
    for b in range(B):
        for h in range(H):
            ref = C.apply_phi(x[b, h], *_sc(kh[b], h, which), variant)[perms[b]]
            assert max_abs_rel(got[b, h], ref) < 1e-5


@pytest.mark.parametrize("d", DS)
def test_k1_small_d_bf16_cache(d):
    B, H, rows, cap, off = 2, 2, 33, 64, 5
    kh, kd = _keys(B, H, d)
    x = C.round_to_format(gauss(4, (B, H, rows, d)), 2)
    perms = [kh[b].span_perm(1, off, rows) for b in range(B)]
    cache = torch.zeros((B, H, cap, d), dtype=torch.bfloat16, device="cuda")
    ops.scramble(dev(x, torch.bfloat16), kd, capi.PHI_INV_T, capi.KEYS_KQ, ops.upload_perms(perms, "cuda"),
                 out=cache, out_row_offset=off)
    got = cache.double().cpu().numpy()
    assert not got[:, :, :off].any() and not got[:, :, off + rows:].any()
    for b in range(B):
        for h in range(H):
            ref = C.round_to_format(C.apply_phi(x[b, h], *_sc(kh[b], h, 0), 1)[perms[b]], 2)
            g = got[b, h, off:off + rows]
            assert (g == ref).mean() > 0.98
            assert np.all(np.abs(g - ref) <= 2.0**-7 * np.abs(ref) + 1e-5 * np.abs(ref).max())


@pytest.mark.parametrize("d", DS)
@pytest.mark.parametrize("kv_dtype", [torch.float32, torch.bfloat16])
def test_k2_small_d_splits_ragged(d, kv_dtype):
    B, Hq, Hkv, lq, cap, S = 3, 4, 2, 3, 700, 3
    fmt = 2 if kv_dtype == torch.bfloat16 else 1
    q = C.round_to_format(gauss(6, (B, Hq, lq, d)), fmt)
    k = C.round_to_format(gauss(7, (B, Hkv, cap, d)), fmt)
    v = C.round_to_format(gauss(8, (B, Hkv, cap, d)), fmt)
    kv_len = np.array([700, 301, 2], np.int32)
    o, st = ops.partial_attention(dev(q, kv_dtype), dev(k, kv_dtype), dev(v, kv_dtype),
                                  torch.from_numpy(kv_len).cuda(), n_splits=S)
    o, st = o.double().cpu().numpy(), st.double().cpu().numpy()
    for b in range(B):
        L = int(kv_len[b])
        chunk = -(-(-(-L // 128)) // S) * 128
        for h in range(Hq):
            for s in range(S):
                a, e = s * chunk, min(L, (s + 1) * chunk)
                if a >= e:
                    assert np.all(st[s, b, h, :, 1] == 0) and np.all(np.isneginf(st[s, b, h, :, 0]))
                    continue
                ro, rm, rs = C.shard_attention(q[b, h], k[b, h // 2, a:e], v[b, h // 2, a:e])
                assert max_abs_rel(o[s, b, h], ro) < 1e-5
                lse = st[s, b, h, :, 0] + np.log(st[s, b, h, :, 1])
                assert np.abs(lse - (rm + np.log(rs))).max() < 1e-5


@pytest.mark.parametrize("d", DS)
def test_k2_small_d_causal(d):
    B, H, lq, L = 1, 2, 20, 20
    q, k, v = gauss(11, (B, H, lq, d)), gauss(12, (B, H, L, d)), gauss(13, (B, H, L, d))
    o, st = ops.partial_attention_causal(dev(q, torch.float32), dev(k, torch.float32), dev(v, torch.float32),
                                         causal_offset=0)
    o = o.double().cpu().numpy()
    for h in range(H):
        ro, rm, rs = C.shard_attention(q[0, h], k[0, h], v[0, h], causal_offset=0)
        assert max_abs_rel(o[0, 0, h], ro) < 1e-5


@pytest.mark.parametrize("d", DS)
def test_k3_small_d_vs_dec_output_merge(d):
    B, H, lq = 2, 3, 5
    srcs, shards = [], [[] for _ in range(B * H)]
    for i, (domain, keyed) in enumerate([(1, True), (2, True), (0, False)]):
        o = gauss(20 + i, (B, H, lq, d))
        m = gauss(30 + i, (B, H, lq)) * 3 + (1000.0 if i == 1 else 0.0)
        s = np.abs(gauss(40 + i, (B, H, lq))) + 0.5
        if i == 2:
            s[0, 0, 2] = 0.0
        kd = pqi = None
        if keyed:
            kh, kd = _keys(B, H, d, domain=domain)
            pq = [kh[b].span_perm(0, 40, lq) for b in range(B)]
            pqi = ops.upload_perms([capi.invert_permutation(p) for p in pq], "cuda")
        srcs.append(ops.MergeSource(dev(o, torch.float32), dev(np.stack([m, s], -1), torch.float32), kd, pqi))
        for b in range(B):
            for h in range(H):
                if keyed:
                    od = C.apply_phi(o[b, h], *_sc(kh[b], h, 1), 2)
                    oo, mm, ss = np.zeros_like(od), np.zeros(lq), np.zeros(lq)
                    oo[pq[b]], mm[pq[b]], ss[pq[b]] = od, m[b, h], s[b, h]
                else:
                    oo, mm, ss = o[b, h], m[b, h], s[b, h]
                shards[b * H + h].append((oo, mm, ss))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    got = ops.unscramble_merge(srcs, err_flag=err).double().cpu().numpy()
    assert int(err.item()) == 0
    for b in range(B):
        for h in range(H):
            sh = shards[b * H + h]
            ref = C.merge_shards([x[0] for x in sh], [x[1] for x in sh], [x[2] for x in sh])
            assert max_abs_rel(got[b, h], ref) < 1e-5


@pytest.mark.parametrize("d", DS)
def test_small_d_end_to_end_fp32(d):
    """The protocol composition at the reference tests' head dims, FP32 mode, vs the oracle and
    vs plain attention (1e-3)."""
    case = Case(B=2, Hq=2, Hkv=2, d=d, lk=40, n_nodes=3, lq=6, dtype=torch.float32, seed=7)
    got = case.run_device(n_splits=2)
    ref, plain = case.oracle(), case.plain()
    assert max_abs_rel(got, ref) < 1e-3 and rel_fro(got, ref) < 1e-3
    assert max_abs_rel(got, plain) < 1e-3 and rel_fro(got, plain) < 1e-3


@pytest.mark.parametrize("d", DS)
def test_small_d_end_to_end_bf16(d):
    case = Case(B=2, Hq=2, Hkv=2, d=d, lk=64, n_nodes=2, lq=1, dtype=torch.bfloat16, seed=8)
    got = case.run_device()
    ref = case.oracle()
    assert max_abs_rel(got, ref) < 2e-2 and rel_fro(got, ref) < 2e-2
