"""K1 on tcgen05 (k1_tc.cu): the GEMM form of scramble + permute must match the oracle's
componentwise apply_phi (rounded once to bf16) and the SIMT FWHT kernel."""
import os

import numpy as np
import pytest
import torch

from oracle import C
from paper_2605_25716_b200 import capi, ops
from tests.gpu_helpers import dev, gauss

pytestmark = pytest.mark.gpu


def _run(x, kd, variant, which, perms, cap, off, simt=False, key_heads=None):
    old = os.environ.get("SDA_K1_SIMT")
    if simt:
        os.environ["SDA_K1_SIMT"] = "1"
    else:
        os.environ.pop("SDA_K1_SIMT", None)
    try:
        B, H, rows, d = x.shape
        out = torch.zeros((B, H, cap, d), dtype=torch.bfloat16, device="cuda")
        ops.scramble(dev(x, torch.bfloat16), kd, variant, which, ops.upload_perms(perms, "cuda"), out=out,
                     out_row_offset=off, key_heads=key_heads)
        torch.cuda.synchronize()
        return out.double().cpu().numpy()
    finally:
        if old is None:
            os.environ.pop("SDA_K1_SIMT", None)
        else:
            os.environ["SDA_K1_SIMT"] = old


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("rows", [128, 300, 1000])
@pytest.mark.parametrize("variant,which", [(capi.PHI_FORWARD, capi.KEYS_KQ), (capi.PHI_INV_T, capi.KEYS_KQ),
                                           (capi.PHI_FORWARD, capi.KEYS_V)])
def test_k1_tc_vs_oracle(d, rows, variant, which):
    B, H, off = 2, 3, 5
    cap = rows + 40
    kh = [capi.negotiate_keyset(capi.shared_seed(1, b + 1), b + 1, 0, 1, H, d) for b in range(B)]
    kd = ops.upload_keys([k.pack() for k in kh], "cuda")
    x = C.round_to_format(gauss(17 + rows, (B, H, rows, d)), 2)
    perms = [kh[b].span_perm(1, off, rows) for b in range(B)]
    got = _run(x, kd, variant, which, perms, cap, off)
    assert not got[:, :, :off].any() and not got[:, :, off + rows:].any()   # never writes outside its rows
    pre = "kq" if which == capi.KEYS_KQ else "v"
    for b in range(B):
        for h in range(H):
            sc = [getattr(kh[b], pre + f)[h] for f in ("_s1", "_p1", "_p2", "_s2")]
            ref = C.round_to_format(C.apply_phi(x[b, h], *sc, variant)[perms[b]], 2)
            g = got[b, h, off:off + rows]
            # one RNE rounding of an f32-accurate value: identical except near bf16 ties (1 ulp),
            # plus absolute f32 accumulation noise on outputs that cancel to ~0
            scale = np.abs(ref).max()
            assert (g == ref).mean() > 0.99
            assert np.all(np.abs(g - ref) <= 2.0**-7 * np.abs(ref) + 1e-5 * scale), np.abs(g - ref).max() / scale


def test_k1_tc_matches_simt_and_gqa():
    B, Hq, Hkv, d, rows = 2, 8, 2, 128, 777
    kh = [capi.negotiate_keyset(capi.shared_seed(1, b + 1), b + 1, 0, 2, Hkv, d) for b in range(B)]
    kd = ops.upload_keys([k.pack() for k in kh], "cuda")
    x = C.round_to_format(gauss(99, (B, Hq, rows, d)), 2)
    perms = [kh[b].span_perm(0, 0, rows) for b in range(B)]
    a = _run(x, kd, capi.PHI_FORWARD, capi.KEYS_KQ, perms, rows, 0, key_heads=Hkv)
    s = _run(x, kd, capi.PHI_FORWARD, capi.KEYS_KQ, perms, rows, 0, simt=True, key_heads=Hkv)
    assert (a == s).mean() > 0.99
    assert np.all(np.abs(a - s) <= 2.0**-7 * np.abs(s) + 1e-5 * np.abs(s).max())


def test_scramble_batch_matches_single_jobs():
    """sda_scramble_batch (three tensor-core jobs sharing one persistent grid: K with phi^-T and
    V with phi into a cache at a row offset, Q with phi into its own buffer, different row counts
    and head counts) is bit-identical to the same three sda_scramble calls."""
    from paper_2605_25716_b200 import capi, ops, protocol
    H, D, L, LQ, CAP = 4, 128, 640, 384, 1024
    keys = protocol.DomainKeys([1, 2], 0, 1, H, D, "cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    kx = torch.randn((2, H, L, D), generator=g, device="cuda").to(torch.bfloat16)
    vx = torch.randn((2, H, L, D), generator=g, device="cuda").to(torch.bfloat16)
    qx = torch.randn((2, 2 * H, LQ, D), generator=g, device="cuda").to(torch.bfloat16)
    pkv, _ = keys.span_perms(1, 100, L)
    pq, _ = keys.span_perms(0, 100 + L, LQ)
    outs = [torch.zeros((2, H, CAP, D), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    outs += [torch.zeros((2, 2 * H, LQ, D), dtype=torch.bfloat16, device="cuda")]
    ref = [t.clone() for t in outs]
    ops.scramble(kx, keys.dev, capi.PHI_INV_T, capi.KEYS_KQ, pkv, out=ref[0], out_row_offset=200, key_heads=H)
    ops.scramble(vx, keys.dev, capi.PHI_FORWARD, capi.KEYS_V, pkv, out=ref[1], out_row_offset=200, key_heads=H)
    ops.scramble(qx, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, pq, out=ref[2], key_heads=H)
    ops.scramble_batch([ops.scramble_job(kx, keys.dev, capi.PHI_INV_T, capi.KEYS_KQ, pkv, out=outs[0], out_row_offset=200, key_heads=H),
                        ops.scramble_job(vx, keys.dev, capi.PHI_FORWARD, capi.KEYS_V, pkv, out=outs[1], out_row_offset=200, key_heads=H),
                        ops.scramble_job(qx, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, pq, out=outs[2], key_heads=H)], D)
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)
