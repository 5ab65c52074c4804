"""Device wire frames (csrc/frame.cu) against the reference's encode_frame / decode_frame /
crc32 (frame.cpp): frame bytes bit-identical for every wire dtype (f64, f32, bf16, f16, quant
2..8) from f64 and f32 device values, special values (+-0, +-inf clamped to the largest finite
bf16 / f16, overflow, subnormals), the parallel CRC on lengths around its 256-byte chunking, the
decoded values equal to values_from_payload, and corrupted / malformed frames rejected."""
import numpy as np
import pytest
import torch

from oracle import C, REF, OracleError
from paper_2605_25716_b200 import capi, ops
from tests.gpu_helpers import gauss

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 4096, 65536 * 3 + 17, (1 << 22) + 5])
def test_crc32_parallel_vs_reference(n):
    rng = np.random.default_rng(n)
    b = rng.integers(0, 256, n, dtype=np.uint8)
    assert ops.crc32(torch.from_numpy(b).cuda()) == REF.crc32(b)


def _values(seed, n, special=False):
    v = C.gaussian(seed, n) * 3.0
    if special:
        v[:12] = [0.0, -0.0, np.inf, -np.inf, 1e39, -3.5e38, 70000.0, 1e-40, -3e-8, 6e-5, 65520.0, 2.0 ** -149]
    return v


@pytest.mark.parametrize("dtype", [0, 1, 2, 3, 18, 19, 22, 24])
@pytest.mark.parametrize("src", [torch.float64, torch.float32])
def test_frame_encode_decode_bit_exact(dtype, src):
    dims = [3, 5, 37]                       # [n_tensors, rows, cols], 555 elements (ragged codes)
    n = int(np.prod(dims))
    special = dtype < 16                    # quantN rejects non-finite values, like the reference
    v = _values(11 + dtype, n, special)
    if src == torch.float32:
        with np.errstate(over="ignore"):
            v = v.astype(np.float32).astype(np.float64)   # the device sees exactly these values
        if special:
            v[4:6] = [np.inf, -np.inf]                # 1e39 / -3.5e38 overflow f32 to inf
    ref = REF.encode_frame(4, 77, 3, 1, 2, dtype, dims, v)
    h = ops.frame_header(4, 77, 3, 1, 2, dtype, dims)
    got = ops.frame_encode(h, torch.from_numpy(v).to(src).cuda()).cpu().numpy()
    assert got.size == ref.size == capi.LIB.sda_frame_bytes(h)
    assert np.array_equal(got, ref), np.nonzero(got != ref)[0][:10]
    # decode the reference's bytes on the device
    hp = ops.frame_parse_header(bytes(ref[:64]), ref.size)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    back = ops.frame_decode(torch.from_numpy(ref).cuda(), hp, torch.float64, err=err).cpu().numpy()
    want = REF.decode_frame(ref, n)
    assert err.item() == 0
    assert np.array_equal(back, want) or np.array_equal(np.isnan(back), np.isnan(want)) and \
        np.array_equal(back[~np.isnan(back)], want[~np.isnan(want)])


def test_frame_corruption_and_malformed_headers():
    dims = [2, 4, 16]
    v = _values(5, 128)
    ref = REF.encode_frame(3, 1, 0, 0, 1, 2, dims, v)
    h = ops.frame_parse_header(bytes(ref[:64]), ref.size)
    bad = ref.copy()
    bad[40] ^= 0x10                                     # one payload bit
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops.frame_decode(torch.from_numpy(bad).cuda(), h, err=err)
    assert err.item() == capi.SDA_ERR_FRAME
    with pytest.raises(OracleError):
        REF.decode_frame(bad, 128)                      # the reference rejects it too (crc mismatch)
    for blob, size in ((b"FATX" + bytes(ref[4:64]), ref.size), (bytes(ref[:64]), ref.size - 1), (bytes(ref[:20]), 20)):
        with pytest.raises(capi.SdaError):
            ops.frame_parse_header(blob, size)


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_wire_round_matches_round_to_format(fmt, dtype):
    """sda_wire_round == the reference's round_to_format (float_format.cpp:26-58) element for
    element: ties, subnormals, overflow and +-inf clamped to +-max_finite, signed zeros."""
    from oracle import REF
    o = REF or C
    x = np.concatenate([gauss(7, (4096,)) * 10.0 ** np.linspace(-40, 40, 4096),
                        [0.0, -0.0, np.inf, -np.inf, 3.4e38, -3.3e38, 1.0 + 2.0**-8, 1.0 + 3 * 2.0**-8,
                         65504.0, 65520.0, 1e-45, 2.0**-130, 1.00390625, 5.960464477539063e-08]])
    x = x.astype(np.float32).astype(np.float64) if dtype == torch.float32 else x
    t = torch.from_numpy(x.copy()).to("cuda").to(dtype)
    ops.wire_round(t, fmt)
    got = t.double().cpu().numpy()
    ref = o.round_to_format(x, fmt)
    if dtype == torch.float32:
        ref = ref.astype(np.float32).astype(np.float64)
    assert np.array_equal(got, ref) and np.array_equal(np.signbit(got), np.signbit(ref))
