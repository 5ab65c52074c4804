"""Generate golden vectors for the hot path FROM THE REFERENCE ITSELF.

Runs the reference's own C++ (compiled in place from /root/reference by oracle/Makefile into
oracle/_ref/libsdattn_ref.so) and stores inputs + outputs in tests/golden/golden.npz. The
fixtures travel with the repo so the GPU box (which has no /root/reference) can pin the oracle
and the CUDA path against reference outputs.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import REF  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    if REF is None:
        raise SystemExit("oracle/_ref/libsdattn_ref.so missing: run `make -C oracle` where /root/reference exists")
    g = {}
    # rng.hpp:20-26 stream + rng.cpp:19-33 gaussians
    for seed in (0, 1, 42, 2**63 + 5):
        g[f"rng_u64_{seed}"] = REF.rng_u64(seed, 16)
        g[f"gauss_{seed}"] = REF.gaussian(seed, 33)
    # rng.cpp:35-39
    tags = [[], [2, 3], [1, 0x7365656B], [5, 2, 1, 1, 0], [2**64 - 1, 0, 7]]
    g["derive_tags"] = np.array([t + [0] * (5 - len(t)) for t in tags], np.uint64)
    g["derive_ntags"] = np.array([len(t) for t in tags], np.int64)
    g["derive_out"] = np.array([REF.derive_seed(99, t) for t in tags], np.uint64)
    # permutation.cpp:29-37
    for n, seed in ((1, 3), (2, 5), (8, 42), (100, 7), (4096, 11)):
        g[f"perm_{n}_{seed}"] = REF.random_permutation(n, seed)
    # negotiate_keyset / span_perm (scrambler.cpp:99-124)
    specs = [(7, 1, 0, 1, 2, 8, 0.125, 8.0, 0), (99, 5, 2, 1, 2, 16, 0.125, 8.0, 0),
             (1234, 3, 1, 4, 3, 64, 0.5, 2.0, 1), (0xABCDEF, 1, 0, 1, 2, 128, 0.125, 8.0, 0)]
    g["ks_specs"] = np.array([s[:6] for s in specs], np.uint64)
    g["ks_mags"] = np.array([[s[6], s[7], s[8]] for s in specs], np.float64)
    for i, s in enumerate(specs):
        ks = REF.negotiate_keyset(*s)
        for k, v in ks.items():
            g[f"ks{i}_{k}"] = np.asarray(v)
        for tag, fp, ln in ((0, 0, 1), (0, 5, 12), (1, 0, 16), (1, 1024, 8), (1, 65536, 257)):
            g[f"ks{i}_span_{tag}_{fp}_{ln}"] = REF.span_perm(ks["token_perm_seed"], tag, fp, ln)
    # float_format.cpp:26-58 incl. the test_tensor.cpp:94-110 KATs
    vals = np.array([0.0, -0.0, 1.0, 1 + 2**-10, 1 + 2**-7, 1 + 3 * 2**-9, 1 + 2**-8, 0.1, 1 / np.sqrt(128), -3.14159,
                     1e-40, 5e-45, 3.4e38, 1e39, -1e39, 65504.0, 65520.0, 1e-5, 6e-8, 2.0**-126, 2.0**-133,
                     np.inf, -np.inf], np.float64)
    rng = np.random.default_rng(5)
    vals = np.concatenate([vals, rng.standard_normal(200) * np.exp(rng.uniform(-30, 30, 200))])
    g["round_in"] = vals
    for fmt in (1, 2, 3):
        g[f"round_out_{fmt}"] = REF.round_to_format(vals, fmt)
    # fwht.cpp:10-26
    for n in (1, 2, 8, 64, 128):
        x = REF.gaussian(100 + n, n)
        g[f"fwht_in_{n}"] = x
        g[f"fwht_out_{n}"] = REF.fwht(x)
    # apply_phi variants (scrambler.cpp:42-85) with keyset-3 head-0 scramblers
    ks = REF.negotiate_keyset(*specs[3])
    x = REF.gaussian(77, 5 * 128).reshape(5, 128)
    g["phi_x"] = x
    for var in (0, 1, 2):
        g[f"phi_out_{var}"] = REF.apply_phi(x, ks["kq_s1"][0], ks["kq_p1"][0], ks["kq_p2"][0], ks["kq_s2"][0], var)
    # shard_attention (attention.cpp:42-78) none + causal
    q = REF.gaussian(1, 6 * 32).reshape(6, 32)
    k = REF.gaussian(2, 9 * 32).reshape(9, 32)
    v = REF.gaussian(3, 9 * 32).reshape(9, 32)
    g["attn_q"], g["attn_k"], g["attn_v"] = q, k, v
    for name, off in (("none", None), ("causal0", 0), ("causal3", 3), ("causalm2", -2)):
        try:
            o, m, s = REF.shard_attention(q, k, v, off)
        except Exception:  # noqa: BLE001 -- all-masked rows are legal for shard_attention
            raise
        g[f"attn_{name}_o"], g[f"attn_{name}_m"], g[f"attn_{name}_s"] = o, m, s
    # merge_shards (attention.cpp:89-123): 3 shards, +1000 logit shift on one
    outs, ms, ss = [], [], []
    for i in range(3):
        o, m, s = REF.shard_attention(q, k[3 * i:3 * i + 3], v[3 * i:3 * i + 3], None)
        if i == 1:
            m = m + 1000.0
        outs.append(o), ms.append(m), ss.append(s)
    g["merge_o"], g["merge_m"], g["merge_s"] = np.stack(outs), np.stack(ms), np.stack(ss)
    g["merge_out"] = REF.merge_shards(outs, ms, ss)
    # full scrambled step composition (protocol path) for 2 nodes, 2 heads, d 64, 1 and 5 query rows
    import ctypes as ct
    lib = REF.lib
    d, lk, nn = 64, 40, 2
    for lq, wire in ((1, 0), (1, 1), (1, 2), (5, 2)):
        qs = REF.gaussian(500 + lq, lq * d).reshape(lq, d)
        ks_ = REF.gaussian(600, nn * lk * d).reshape(nn, lk, d)
        vs_ = REF.gaussian(700, nn * lk * d).reshape(nn, lk, d)
        out = np.zeros((lq, d))
        P = ct.POINTER(ct.c_double)
        rc = lib.ref_scrambled_step(ct.c_uint64(7), ct.c_uint64(1), ct.c_uint32(0), ct.c_size_t(2), ct.c_size_t(1),
                                    ct.c_size_t(d), ct.c_double(0.125), ct.c_double(8.0), ct.c_int(0),
                                    ct.c_int(wire), ct.c_size_t(nn), qs.ctypes.data_as(P), ct.c_size_t(lq),
                                    ct.c_uint64(nn * lk), ks_.ctypes.data_as(P), vs_.ctypes.data_as(P),
                                    ct.c_size_t(lk), out.ctypes.data_as(P))
        assert rc == 0
        g[f"step_{lq}_{wire}_q"], g[f"step_{lq}_{wire}_k"], g[f"step_{lq}_{wire}_v"] = qs, ks_, vs_
        g[f"step_{lq}_{wire}_out"] = out
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
