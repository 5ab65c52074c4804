"""Wire frame pins (frame.cpp): the oracle's CRC-32 against the reference's and the standard
check value, and the reference's own frame round trip used by the device tests."""
import numpy as np

from oracle import C, REF


def test_crc32_known_answer_and_random():
    assert C.crc32(np.frombuffer(b"123456789", np.uint8)) == 0xCBF43926 == REF.crc32(np.frombuffer(b"123456789", np.uint8))
    rng = np.random.default_rng(3)
    for n in (0, 1, 3, 255, 256, 257, 4099):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert C.crc32(b) == REF.crc32(b)


def test_reference_frame_roundtrip_and_layout():
    v = C.gaussian(5, 2 * 3 * 8)
    f = REF.encode_frame(3, 0x0102030405060708, 2, 1, 4, 2, [2, 3, 8], v)
    assert bytes(f[:4]) == b"FATN" and f[4] == 1 and f[5] == 3 and f[20] == 2
    assert len(f) == 25 + 4 * 3 + 2 * 48 + 4
    assert REF.crc32(f[:-4]) == int.from_bytes(bytes(f[-4:]), "little")
    back = REF.decode_frame(f, 48)
    assert np.allclose(back, v, rtol=1e-2, atol=1e-30)          # bf16 payload
