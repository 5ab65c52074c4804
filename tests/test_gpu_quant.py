"""Device quantised wire (csrc/quant.cu) against the reference's quantize_affine / dequantize:
codes, scale and zero point bit-exact on the same input values (f64, f32 and bf16 inputs, the
latter two exactly representable in f64), dequantised values bit-exact, the in-place round trip
equal to dequantize(quantize(x)) per tensor, and the non-finite error flag."""
import numpy as np
import pytest
import torch

from oracle import REF
from paper_2605_25716_b200 import capi, ops

pytestmark = pytest.mark.gpu


def _tensors(seed, n, count, scale=2.0):
    from oracle import C
    x = C.gaussian(seed, n * count).reshape(n, count) * scale
    x[0] += 10.0                       # different ranges per tensor
    if n > 2:
        x[2] = 0.75                    # a constant tensor
    return x


@pytest.mark.parametrize("bits", [2, 3, 5, 8])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16])
def test_quantize_affine_bit_exact(bits, dtype):
    n, count = 5, 1003                  # ragged: codes straddle bytes and the last group is partial
    x = torch.from_numpy(_tensors(7 + bits, n, count)).to(dtype).cuda()
    codes, sc, zp = ops.quantize_affine(x, bits)
    deq = ops.dequantize(codes, sc, zp, count, bits)
    xr = ops.quant_roundtrip(x.double().clone(), bits)
    torch.cuda.synchronize()
    xh = x.double().cpu().numpy()
    for t in range(n):
        c_ref, s_ref, z_ref = REF.quantize_affine(xh[t], bits)
        assert np.array_equal(codes[t].cpu().numpy(), c_ref), t
        assert sc[t].item() == s_ref and zp[t].item() == z_ref, t
        d_ref = REF.dequantize(c_ref, count, bits, s_ref, z_ref)
        assert np.array_equal(deq[t].cpu().numpy(), d_ref), t
        assert np.array_equal(xr[t].cpu().numpy(), d_ref), t


def test_roundtrip_f32_in_place_and_errors():
    x = torch.from_numpy(_tensors(3, 4, 640)).float().cuda()
    xs = x.double().cpu().numpy()
    ops.quant_roundtrip(x, 6)
    for t in range(4):
        c, s, z = REF.quantize_affine(xs[t], 6)
        assert np.array_equal(x[t].cpu().numpy(), REF.dequantize(c, 640, 6, s, z).astype(np.float32))
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    bad = torch.ones((2, 16), dtype=torch.float32, device="cuda")
    bad[1, 3] = float("nan")
    ops.quantize_affine(bad, 8, err=err)
    assert err.item() == 1   # SDA_ERR_INVALID_ARGUMENT (quant.cpp:35 throws std::invalid_argument)
    with pytest.raises(Exception):
        ops.quantize_affine(bad, 9)


# --- the quantised wire inside K1 / K3 ------------------------------------------
def _keys(B, H, d, domain=1):
    kh = [capi.negotiate_keyset(capi.shared_seed(1, b + 1), b + 1, 0, domain, H, d) for b in range(B)]
    return kh, ops.upload_keys([k.pack() for k in kh], "cuda")


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("rows", [1, 77])
@pytest.mark.parametrize("variant,which", [(capi.PHI_FORWARD, capi.KEYS_KQ), (capi.PHI_INV_T, capi.KEYS_KQ),
                                           (capi.PHI_FORWARD, capi.KEYS_V)])
def test_k1_quant_epilogue_equals_scramble_then_roundtrip(bits, rows, variant, which):
    """sda_scramble_quant (min / max pass + quantising epilogue) == sda_scramble to f32 followed by
    sda_quant_roundtrip per (request, head) tensor -- bit for bit: the same f32 scrambled values
    meet the same bit-exact quantiser (test_quantize_affine_bit_exact)."""
    B, H, d = 3, 4, 64
    from oracle import C
    kh, kd = _keys(B, H, d)
    x = torch.from_numpy(C.gaussian(90 + rows, B * H * rows * d).reshape(B, H, rows, d)).float().cuda()
    perm = ops.upload_perms([kh[b].span_perm(1, 3 * b, rows) for b in range(B)], "cuda")
    fused = ops.scramble_quant(x, kd, variant, which, bits, perm)
    plain = ops.scramble(x, kd, variant, which, perm, out_dtype=torch.float32)
    ref = ops.quant_roundtrip(plain.reshape(B * H, rows * d).contiguous(), bits).reshape(B, H, rows, d)
    torch.cuda.synchronize()
    assert torch.equal(fused, ref)
    # and the wire really is quantised: at most 2^bits distinct values per tensor
    for b in range(B):
        assert torch.unique(fused[b, 0]).numel() <= 2 ** bits


def test_k1_quant_nonfinite_sets_err():
    B, H, d = 1, 2, 32
    kh, kd = _keys(B, H, d)
    x = torch.randn((B, H, 5, d), device="cuda")
    x[0, 1, 2, 3] = float("inf")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops.scramble_quant(x, kd, capi.PHI_FORWARD, capi.KEYS_KQ, 8, err=err)
    assert int(err.item()) == 1   # SDA_ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("lq", [1, 50])
def test_k3_quant_input_path(bits, lq):
    """sda_unscramble_merge_quant: each domain's O' (its splits folded, normalised, still
    scrambled) goes through dequantize(quantize_affine(.)) before its unscramble. Against the same
    steps done separately: fold each domain's splits with K3 (plaintext merge), quant round trip
    per (request, head) tensor, then K3 over the quantised domain partials."""
    from oracle import C
    B, H, d = 2, 3, 128
    srcs, groups = [], []
    for dom in range(2):
        kh, kd = _keys(B, H, d, domain=dom + 1)
        pq = [kh[b].span_perm(0, 11, lq) for b in range(B)]
        pqi = ops.upload_perms([capi.invert_permutation(p) for p in pq], "cuda") if lq > 1 else None
        gs = []
        for s in range(3):
            o = torch.from_numpy(C.gaussian(200 + 10 * dom + s, B * H * lq * d).reshape(B, H, lq, d)).float().cuda()
            m = torch.from_numpy(C.gaussian(300 + 10 * dom + s, B * H * lq).reshape(B, H, lq)).float().cuda() * 2
            ssum = torch.rand((B, H, lq), device="cuda") + 0.5
            st = torch.stack([m, ssum], -1).contiguous()
            srcs.append(ops.MergeSource(o, st, kd, pqi))
            gs.append((o, st))
        groups.append((gs, kd, pqi))
    got = ops.unscramble_merge(srcs, quant_bits=bits)
    # the separate form: fold (plaintext merge of the splits, stats out), round trip, merge
    folded = []
    for gs, kd, pqi in groups:
        fo = torch.empty((B, H, lq, d), device="cuda")
        fst = torch.empty((B, H, lq, 2), device="cuda")
        ops.unscramble_merge([ops.MergeSource(o, st) for o, st in gs], out=fo, out_stats=fst)
        ops.quant_roundtrip(fo.reshape(B * H, lq * d), bits)
        folded.append(ops.MergeSource(fo, fst, kd, pqi))
    ref = ops.unscramble_merge(folded)
    torch.cuda.synchronize()
    # the fused form divides the fold by its weight in f32 inside K3: the few values on a code
    # boundary can land one quantisation step away, so compare against the step size
    step = (ref.abs().amax() * 2 / (2 ** bits - 1)).item()
    diff = (got - ref).abs()
    assert diff.max().item() <= 1.01 * step
    assert (diff > 1e-4 * ref.abs().amax()).float().mean().item() < 0.02
