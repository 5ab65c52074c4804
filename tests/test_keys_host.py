"""Product host key derivation (libsdattn_b200.so, CPU code) is bit-exact with the oracle."""
import numpy as np
import pytest

from oracle import C
from paper_2605_25716_b200 import capi


def test_seed_and_perm():
    assert capi.shared_seed(1, 1) == C.derive_seed(1, [1, 0x7365656B])
    assert capi.derive_seed(99, [5, 2, 1]) == C.derive_seed(99, [5, 2, 1])
    for n, seed in ((1, 1), (8, 42), (1000, 9)):
        assert np.array_equal(capi.random_permutation(n, seed), C.random_permutation(n, seed))


def test_negotiate_keyset_bit_exact_many_specs():
    rng = np.random.default_rng(10)
    for i in range(400):
        d = int(2 ** rng.integers(0, 9))
        h = int(rng.integers(1, 5))
        spec = (int(rng.integers(0, 2**63)), int(rng.integers(0, 1 << 40)), int(rng.integers(0, 80)),
                int(rng.integers(0, 9)), h, d)
        lo, hi = (0.125, 8.0) if i % 3 else (float(rng.uniform(0.1, 1)), float(rng.uniform(1, 10)))
        mode = i % 2
        a = capi.negotiate_keyset(*spec, mag_lo=lo, mag_hi=hi, mode=mode)
        b = C.negotiate_keyset(*spec, lo, hi, mode)
        for f in capi.HostKeyset.FIELDS_F + capi.HostKeyset.FIELDS_U:
            assert np.array_equal(getattr(a, f), b[f]), f
        assert a.token_perm_seed == b["token_perm_seed"]
        n = int(rng.integers(1, 5000))
        fp = int(rng.integers(0, 1 << 30))
        assert np.array_equal(a.span_perm(1, fp, n), C.span_perm(b["token_perm_seed"], 1, fp, n))


def test_pack_layout():
    d, H = 64, 2
    ks = capi.negotiate_keyset(capi.shared_seed(1, 3), 3, 0, 1, H, d)
    img = ks.pack()
    assert img.size == capi.keyset_bytes(H, d) == H * 68 * d
    for h in range(H):
        for which, pre in ((0, "kq"), (1, "v")):
            base = h * 68 * d + which * 34 * d
            f = img[base:base + 24 * d].view(np.float32).reshape(6, d)
            u = img[base + 24 * d:base + 32 * d].view(np.uint16).reshape(4, d)
            s1, s2 = getattr(ks, pre + "_s1")[h], getattr(ks, pre + "_s2")[h]
            p1, p2 = getattr(ks, pre + "_p1")[h], getattr(ks, pre + "_p2")[h]
            r = 1 / np.sqrt(d)
            np.testing.assert_array_equal(f[0], s1.astype(np.float32))
            np.testing.assert_array_equal(f[1], (1 / s1).astype(np.float32))
            np.testing.assert_array_equal(f[2], (s2 * r).astype(np.float32))
            np.testing.assert_array_equal(f[3], (r / s2).astype(np.float32))
            np.testing.assert_array_equal(f[4], (1 / s2).astype(np.float32))
            np.testing.assert_array_equal(f[5], (r / s1).astype(np.float32))
            assert np.array_equal(u[0], p1) and np.array_equal(u[1], p2)
            assert np.array_equal(u[2][p1], np.arange(d)) and np.array_equal(u[3][p2], np.arange(d))


@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_pack_gather_schedules_are_bank_conflict_free(d):
    """The u8 gather schedules of the key image (sdattn_internal.h kSched*): in every one of the
    E = d/32 loads of a warp-wide gather through P2 (resp. P1), the 32 lanes' addresses fall in 32
    different shared-memory banks, and each lane takes each of its E elements exactly once."""
    H, E = 3, d // 32
    ks = capi.negotiate_keyset(capi.shared_seed(1, 9), 9, 2, 4, H, d)
    img = ks.pack()
    for h in range(H):
        for which in (0, 1):
            base = h * 68 * d + which * 34 * d
            u = img[base + 24 * d:base + 32 * d].view(np.uint16).reshape(4, d)
            sch = img[base + 32 * d:base + 34 * d].reshape(2, d)
            for tab, q in ((0, u[1]), (1, u[0])):   # schedule 0 gathers through P2, 1 through P1
                order = sch[tab].reshape(32, E)
                assert all(sorted(order[l].tolist()) == list(range(E)) for l in range(32))
                for k in range(E):
                    assert len({int(q[l * E + order[l, k]]) % 32 for l in range(32)}) == 32, (h, which, tab, k)


def test_invert_permutation():
    p = capi.random_permutation(777, 5)
    inv = capi.invert_permutation(p)
    assert np.array_equal(inv[p], np.arange(777))
