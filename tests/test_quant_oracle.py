"""The quantised wire (quant.cpp:26-67): the oracle's C restatement against the reference's own
quantize_affine / dequantize, bit for bit, over bit widths 2..8, ragged counts (not multiples of
8, codes straddling bytes), constant and empty tensors, and the error cases."""
import numpy as np
import pytest

from oracle import C, REF, OracleError


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("n", [0, 1, 7, 9, 64, 1001])
def test_quantize_dequantize_oracle_vs_reference(bits, n):
    v = C.gaussian(1000 + 10 * bits + n, max(n, 1))[:n] * 3.0 + 0.5
    c0, s0, z0 = C.quantize_affine(v, bits)
    c1, s1, z1 = REF.quantize_affine(v, bits)
    assert np.array_equal(c0, c1) and s0 == s1 and z0 == z1
    assert np.array_equal(C.dequantize(c0, n, bits, s0, z0), REF.dequantize(c1, n, bits, s1, z1))


def test_constant_tensor_and_rounding_ties():
    c, s, z = REF.quantize_affine(np.full(13, 2.5), 4)
    assert s == 0.0 and z == 2.5 and not c.any()                # constant: scale 0, all codes 0
    v = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0])           # exact half-steps: nearbyint ties to even
    for lib in (C, REF):
        c, s, z = lib.quantize_affine(v, 2)
        assert s == 1.0 and z == 0.0
        assert np.array_equal(lib.dequantize(c, v.size, 2, s, z), [0, 0, 1, 2, 2, 2, 3])


def test_errors():
    for lib in (C, REF):
        with pytest.raises(OracleError):
            lib.quantize_affine(np.array([1.0, np.inf]), 8)
        with pytest.raises(OracleError):
            lib.quantize_affine(np.array([1.0, 2.0]), 9)
