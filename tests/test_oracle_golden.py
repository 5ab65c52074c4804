"""The C restatement (oracle/sdattn_oracle.c) against golden vectors produced by the reference
itself (tests/golden/make_golden.py) and against the reference's own known-answer tests."""
import os

import numpy as np
import pytest

from oracle import C

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_rng_stream_and_gaussians():
    for seed in (0, 1, 42, 2**63 + 5):
        assert np.array_equal(C.rng_u64(seed, 16), G[f"rng_u64_{seed}"])
        assert np.array_equal(C.gaussian(seed, 33), G[f"gauss_{seed}"])  # bitwise: same libm


def test_rng_kat_appendix_a():
    # SURVEY Appendix A (the survey printed the three draws in reverse argument-evaluation order)
    assert [hex(x) for x in C.rng_u64(1, 3)] == ["0x910a2dec89025cc1", "0xbeeb8da1658eec67", "0xf893a2eefb32555e"]
    assert C.derive_seed(1, [2, 3]) == 0x3A809B8E075FBE92
    assert C.derive_seed(1, [1, 0x7365656B]) == 0x0CDDAB0D83EE9276


def test_derive_seed():
    for tags, n, want in zip(G["derive_tags"], G["derive_ntags"], G["derive_out"]):
        assert C.derive_seed(99, list(tags[:n])) == int(want)


def test_random_permutation():
    for n, seed in ((1, 3), (2, 5), (8, 42), (100, 7), (4096, 11)):
        assert np.array_equal(C.random_permutation(n, seed), G[f"perm_{n}_{seed}"])
    assert list(C.random_permutation(8, 42)) == [3, 1, 6, 2, 4, 0, 7, 5]  # Appendix A


def test_keysets_and_span_perms():
    for i, (spec, mags) in enumerate(zip(G["ks_specs"], G["ks_mags"])):
        ks = C.negotiate_keyset(int(spec[0]), int(spec[1]), int(spec[2]), int(spec[3]), int(spec[4]), int(spec[5]),
                                float(mags[0]), float(mags[1]), int(mags[2]))
        for k in ("kq_s1", "kq_p1", "kq_p2", "kq_s2", "v_s1", "v_p1", "v_p2", "v_s2"):
            assert np.array_equal(ks[k], G[f"ks{i}_{k}"]), k  # bit-exact, f64 included
        assert ks["token_perm_seed"] == int(G[f"ks{i}_token_perm_seed"])
        for tag, fp, ln in ((0, 0, 1), (0, 5, 12), (1, 0, 16), (1, 1024, 8), (1, 65536, 257)):
            assert np.array_equal(C.span_perm(ks["token_perm_seed"], tag, fp, ln), G[f"ks{i}_span_{tag}_{fp}_{ln}"])


def test_keyset_kat_appendix_a():
    ks = C.negotiate_keyset(7, 1, 0, 1, 2, 8)
    assert ks["token_perm_seed"] == 0x31FD1DD13369A17D
    assert list(C.span_perm(ks["token_perm_seed"], 1, 0, 16)) == [10, 1, 2, 3, 8, 4, 13, 14, 9, 11, 5, 12, 6, 7, 15, 0]
    assert list(ks["kq_p1"][0]) == [3, 1, 4, 5, 7, 6, 0, 2]
    assert list(ks["kq_p2"][0]) == [4, 3, 6, 5, 1, 7, 2, 0]
    assert ks["kq_s1"][0][0] == -1.2972935968595196
    assert ks["v_s2"][1][0] == 7.4115493689699017
    assert list(C.span_perm(ks["token_perm_seed"], 1, 1024, 8)) == [3, 2, 6, 0, 4, 1, 7, 5]
    # a single-row span gets the identity
    assert list(C.span_perm(ks["token_perm_seed"], 0, 77, 1)) == [0]


def test_round_to_format():
    for fmt in (1, 2, 3):
        got = C.round_to_format(G["round_in"], fmt)
        assert np.array_equal(got, G[f"round_out_{fmt}"], equal_nan=True), fmt
    # test_tensor.cpp:94-100 bf16 KATs
    r = C.round_to_format(np.array([1 + 2**-10, 1 + 2**-7, 1 + 2**-8, 1 + 3 * 2**-8, 0.1]), 2)
    assert list(r) == [1.0, 1.0078125, 1.0, 1 + 4 * 2**-8, 0.10009765625]


def test_fwht():
    for n in (1, 2, 8, 64, 128):
        assert np.array_equal(C.fwht(G[f"fwht_in_{n}"]), G[f"fwht_out_{n}"])
    # test_tensor.cpp:135-158 flavoured: unit impulse -> constant 1/sqrt(n); involution
    x = np.zeros(16)
    x[0] = 1
    assert np.allclose(C.fwht(x), 0.25)
    y = np.random.default_rng(0).standard_normal(64)
    assert np.allclose(C.fwht(C.fwht(y)), y, atol=1e-12)


def test_apply_phi():
    ks = C.negotiate_keyset(0xABCDEF, 1, 0, 1, 2, 128)
    for var in (0, 1, 2):
        got = C.apply_phi(G["phi_x"], ks["kq_s1"][0], ks["kq_p1"][0], ks["kq_p2"][0], ks["kq_s2"][0], var)
        assert np.array_equal(got, G[f"phi_out_{var}"]), var


def test_shard_attention_and_merge():
    for name, off in (("none", None), ("causal0", 0), ("causal3", 3), ("causalm2", -2)):
        o, m, s = C.shard_attention(G["attn_q"], G["attn_k"], G["attn_v"], off)
        assert np.array_equal(o, G[f"attn_{name}_o"])
        assert np.array_equal(m, G[f"attn_{name}_m"])
        assert np.array_equal(s, G[f"attn_{name}_s"])
    got = C.merge_shards(list(G["merge_o"]), list(G["merge_m"]), list(G["merge_s"]))
    assert np.array_equal(got, G["merge_out"])


def test_merge_errors():
    o = np.ones((2, 4))
    with pytest.raises(Exception):
        C.merge_shards([], [], [])
    with pytest.raises(Exception):
        C.merge_shards([o, o], [np.zeros(2), np.zeros(2)], [np.array([0.0, 1.0]), np.array([0.0, 1.0])])
    # single shard is returned verbatim (attention.cpp:97-101)
    x = np.random.default_rng(1).standard_normal((2, 4))
    assert np.array_equal(C.merge_shards([x], [np.zeros(2)], [np.ones(2)]), x)


def test_scrambled_step_composition():
    # the C restatement composed like the protocol == the reference's own composition
    for lq, wire in ((1, 0), (1, 1), (1, 2), (5, 2)):
        q, k, v = G[f"step_{lq}_{wire}_q"], G[f"step_{lq}_{wire}_k"], G[f"step_{lq}_{wire}_v"]
        got = C.scrambled_step(7, 1, 0, 2, 1, q, 80, list(k), list(v), wire_fmt=wire)
        assert np.array_equal(got, G[f"step_{lq}_{wire}_out"]), (lq, wire)
        # and equals plain attention over the concatenated context (exact in f64 up to 1e-8)
        if wire == 0:
            plain, _, _ = C.shard_attention(q, np.concatenate(list(k)), np.concatenate(list(v)))
            assert np.abs(got - plain).max() < 1e-8
