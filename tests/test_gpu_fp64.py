"""FP64 mode (SDA_F64): the reference's f64 arithmetic in its own operation order on the device
(f64_path.cu). K1 is bit-identical to the reference's apply_phi / apply_phi_inv_t / apply_phi_inv
(oracle/_ref, the reference compiled from its own sources); K2's logits and row_max are
bit-identical to shard_attention's, its exp-weighted sums agree to ~1e-15 (CUDA exp vs glibc exp);
the composed path matches the oracle and plain attention to 1e-12."""
import numpy as np
import pytest
import torch

from oracle import C, REF
from paper_2605_25716_b200 import capi, ops
from tests.gpu_helpers import Case, gauss, max_abs_rel, rel_fro

pytestmark = pytest.mark.gpu
O = REF or C   # the reference itself when it was built here (bitwise equal to C on every golden vector)
DS = [4, 8, 16, 32, 64, 128, 256]


def _keys(B, H, d, domain=1):
    kh = [capi.negotiate_keyset(capi.shared_seed(1, b + 1), b + 1, 0, domain, H, d) for b in range(B)]
    return kh, ops.upload_keys([k.pack_f64() for k in kh], "cuda")


def _sc(ks, h, which):
    p = "kq" if which == 0 else "v"
    return (getattr(ks, p + "_s1")[h], getattr(ks, p + "_p1")[h], getattr(ks, p + "_p2")[h], getattr(ks, p + "_s2")[h])


def _d(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda")


@pytest.mark.parametrize("d", DS)
@pytest.mark.parametrize("variant,which", [(capi.PHI_FORWARD, capi.KEYS_KQ), (capi.PHI_INV_T, capi.KEYS_KQ),
                                           (capi.PHI_FORWARD, capi.KEYS_V)])
def test_k1_f64_bit_exact(d, variant, which):
    B, H, rows = 2, 2, 33
    kh, kd = _keys(B, H, d)
    x = gauss(3, (B, H, rows, d)) * 3.0
    perms = [kh[b].span_perm(1, 5 * b, rows) for b in range(B)]
    got = ops.scramble(_d(x), kd, variant, which, ops.upload_perms(perms, "cuda")).cpu().numpy()
    for b in range(B):
        for h in range(H):
            ref = O.apply_phi(x[b, h], *_sc(kh[b], h, which), variant)[perms[b]]
            assert np.array_equal(got[b, h], ref), (b, h, np.abs(got[b, h] - ref).max())


@pytest.mark.parametrize("d", [16, 64, 128])
def test_k3_f64_dec_output_bit_exact_single_source(d):
    """dec_output alone (one keyed source): apply_phi_inv + the p_q scatter, bit-exact."""
    B, H, lq = 2, 2, 9
    kh, kd = _keys(B, H, d, domain=2)
    o = gauss(20, (B, H, lq, d))
    st = np.stack([gauss(21, (B, H, lq)), np.abs(gauss(22, (B, H, lq))) + 0.5], -1)
    pq = [kh[b].span_perm(0, 40, lq) for b in range(B)]
    pqi = ops.upload_perms([capi.invert_permutation(p) for p in pq], "cuda")
    out_st = torch.empty((B, H, lq, 2), dtype=torch.float64, device="cuda")
    got = ops.unscramble_merge([ops.MergeSource(_d(o), _d(st), kd, pqi)], out_dtype=torch.float64,
                               out_stats=out_st).cpu().numpy()
    gst = out_st.cpu().numpy()
    for b in range(B):
        for h in range(H):
            od = O.apply_phi(o[b, h], *_sc(kh[b], h, 1), 2)
            ref, rst = np.zeros_like(od), np.zeros((lq, 2))
            ref[pq[b]], rst[pq[b]] = od, st[b, h]
            assert np.array_equal(got[b, h], ref) and np.array_equal(gst[b, h], rst)


@pytest.mark.parametrize("d", [8, 64, 128])
def test_k2_f64_vs_shard_attention(d):
    B, Hq, Hkv, lq, cap, S = 2, 4, 2, 3, 500, 2
    q, k, v = gauss(6, (B, Hq, lq, d)), gauss(7, (B, Hkv, cap, d)), gauss(8, (B, Hkv, cap, d))
    kv_len = np.array([500, 77], np.int32)
    o, st = ops.partial_attention(_d(q), _d(k), _d(v), torch.from_numpy(kv_len).cuda(), n_splits=S)
    assert o.dtype == torch.float64
    o, st = o.cpu().numpy(), st.cpu().numpy()
    for b in range(B):
        L = int(kv_len[b])
        chunk = -(-(-(-L // 128)) // S) * 128
        for h in range(Hq):
            for s in range(S):
                a, e = s * chunk, min(L, (s + 1) * chunk)
                if a >= e:
                    assert np.all(st[s, b, h, :, 1] == 0)
                    continue
                ro, rm, rs = O.shard_attention(q[b, h], k[b, h // 2, a:e], v[b, h // 2, a:e])
                assert np.array_equal(st[s, b, h, :, 0], rm)          # logits bit-exact
                assert np.allclose(st[s, b, h, :, 1], rs, rtol=1e-14, atol=0)
                assert max_abs_rel(o[s, b, h], ro) < 1e-14


def test_k2_f64_causal_and_k3_merge():
    lq, lk, d = 7, 10, 16
    q, k, v = gauss(61, (1, 2, lq, d)), gauss(62, (1, 2, lk, d)), gauss(63, (1, 2, lk, d))
    o, st = ops.partial_attention_causal(_d(q), _d(k), _d(v), causal_offset=-2)
    o, st = o.cpu().numpy()[0, 0], st.cpu().numpy()[0, 0]
    for h in range(2):
        ro, rm, rs = O.shard_attention(q[0, h], k[0, h], v[0, h], -2)
        live = rs > 0
        assert np.array_equal(st[h, :, 1] > 0, live)
        assert np.allclose(o[h][live], ro[live], rtol=1e-14, atol=1e-15)
    # merge_shards over plaintext sources, +1000 shift
    B, H, lq = 1, 2, 4
    srcs, outs, ms, ss = [], [], [], []
    for i in range(3):
        oo = gauss(70 + i, (B, H, lq, d))
        m = gauss(80 + i, (B, H, lq)) + (1000.0 if i == 1 else 0.0)
        s = np.abs(gauss(90 + i, (B, H, lq))) + 0.1
        srcs.append(ops.MergeSource(_d(oo), _d(np.stack([m, s], -1))))
        outs.append(oo), ms.append(m), ss.append(s)
    got = ops.unscramble_merge(srcs, out_dtype=torch.float64).cpu().numpy()
    for h in range(H):
        ref = O.merge_shards([x[0, h] for x in outs], [x[0, h] for x in ms], [x[0, h] for x in ss])
        assert max_abs_rel(got[0, h], ref) < 1e-14


@pytest.mark.parametrize("d,lq", [(16, 6), (64, 1), (128, 5)])
def test_fp64_mode_end_to_end(d, lq):
    """The protocol composition in the FP64 mode: the oracle at wire f64 and plain attention, 1e-12."""
    case = Case(B=2, Hq=2, Hkv=2, d=d, lk=96, n_nodes=3, lq=lq, dtype=torch.float64, seed=13)
    got = case.run_device(n_splits=2, out_dtype=torch.float64)
    ref, plain = case.oracle(), case.plain()
    assert max_abs_rel(got, ref) < 1e-12 and rel_fro(got, ref) < 1e-12
    assert max_abs_rel(got, plain) < 1e-12
