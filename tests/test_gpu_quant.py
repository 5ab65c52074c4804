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
