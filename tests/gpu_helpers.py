"""Shared helpers for the GPU parity tests: seeded synthetic inputs (the reference's own
Box-Muller stream), the device pipeline, and the rounding-matched oracle."""
from __future__ import annotations

import numpy as np
import torch

from oracle import C, FMT_BF16, FMT_F32, max_abs_rel, rel_fro
from paper_2605_25716_b200 import protocol

__all__ = ["gauss", "dev", "Case", "max_abs_rel", "rel_fro", "FMT_BF16", "FMT_F32", "assert_lse", "LSE_TOL"]

# SURVEY 8(d) metric 4: LSE = row_max + ln(exp_sum) against the rounding-matched oracle (both
# sides see identical bf16 / f32 Q', K', V', so only the accumulation order differs)
LSE_TOL = {"bf16": 1e-3, "f32": 1e-5}


def assert_lse(st, rm, rs, tol, what=""):
    """st [..., 2] = device (row_max, exp_sum); rm, rs = the oracle's. Masked rows (exp_sum 0)
    must be masked on both sides; elsewhere |LSE_dev - LSE_ref| <= tol (absolute, natural log)."""
    st = np.asarray(st, np.float64)
    rm, rs = np.asarray(rm, np.float64), np.asarray(rs, np.float64)
    dead = rs == 0
    assert np.array_equal(st[..., 1] == 0, dead), ("masked rows differ", what)
    live = ~dead
    if live.any():
        got = st[..., 0][live] + np.log(st[..., 1][live])
        ref = rm[live] + np.log(rs[live])
        err = float(np.abs(got - ref).max())
        assert err <= tol, (f"LSE off by {err:.3e} > {tol:.0e}", what)


def gauss(seed: int, shape) -> np.ndarray:
    n = int(np.prod(shape))
    return C.gaussian(seed, n).reshape(shape)


def dev(x: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(dtype)


class Case:
    """B requests x Hq q-heads (Hkv kv-heads) x d; n_nodes domains with lk keys each; lq query
    rows at q_first_pos = n_nodes * lk. Inputs are rounded to the storage dtype so the device and
    the oracle see identical plaintext values."""

    def __init__(self, B, Hq, Hkv, d, lk, n_nodes, lq=1, dtype=torch.bfloat16, seed=1, master_seed=1,
                 q_scale=1.0, kv_lens=None, mag=(0.125, 8.0), mode=0):
        self.B, self.Hq, self.Hkv, self.d, self.lk, self.n, self.lq = B, Hq, Hkv, d, lk, n_nodes, lq
        self.dtype = dtype
        self.fmt = {torch.bfloat16: FMT_BF16, torch.float32: FMT_F32, torch.float64: 0}[dtype]
        self.master = master_seed
        self.mag, self.mode = mag, mode
        self.kv_lens = kv_lens  # optional per-node list of per-request lengths (<= lk)
        rnd = lambda s, shp: C.round_to_format(gauss(s, shp), self.fmt)  # noqa: E731
        self.q = rnd(seed, (B, Hq, lq, d)) * q_scale
        self.q = C.round_to_format(self.q, self.fmt)
        self.k = [rnd(seed + 10 + 2 * i, (B, Hkv, lk, d)) for i in range(n_nodes)]
        self.v = [rnd(seed + 11 + 2 * i, (B, Hkv, lk, d)) for i in range(n_nodes)]
        self.q_first_pos = n_nodes * lk

    def request_ids(self):
        return [b + 1 for b in range(self.B)]

    def run_device(self, n_splits=None, out_dtype=torch.float32, wrong_keys_at_finish=False):
        domains = []
        for i in range(self.n):
            keys = protocol.DomainKeys(self.request_ids(), 0, i + 1, self.Hkv, self.d, "cuda", self.master,
                                       self.mag[0], self.mag[1], self.mode, fp64=self.dtype == torch.float64)
            shard = protocol.KVShard(self.B, self.Hkv, self.lk, self.d, "cuda", self.dtype)
            shard.ship_segment(dev(self.k[i], self.dtype), dev(self.v[i], self.dtype), keys, first_pos=i * self.lk)
            domains.append((keys, shard))
        q = dev(self.q, self.dtype)
        if not wrong_keys_at_finish:
            out = protocol.scrambled_attention(q, domains, self.q_first_pos, n_splits=n_splits, out_dtype=out_dtype)
        else:
            partials = []
            for keys, shard in domains:
                q_s, pinv = keys.scramble_q(q, self.q_first_pos, out_dtype=shard.k.dtype)
                o, st = shard.serve(q_s, n_splits=n_splits)
                bad = protocol.DomainKeys(self.request_ids(), 0, keys.domain, self.Hkv, self.d, "cuda",
                                          self.master ^ 0xDEADBEEF, fp64=self.dtype == torch.float64)  # protocol.cpp:232-243 sabotage
                partials.append((o, st, bad, pinv))
            out = protocol.finish(partials, out_dtype=out_dtype, kv_heads=self.Hkv)
        torch.cuda.synchronize()
        return out.double().cpu().numpy()

    def oracle(self, pairs=None):
        """Rounding-matched reference composition (Q', K', V' rounded to the storage format)."""
        G = self.Hq // self.Hkv
        out = np.zeros_like(self.q)
        pairs = pairs or [(b, h) for b in range(self.B) for h in range(self.Hq)]
        for b, h in pairs:
            ss = C.derive_seed(self.master, [b + 1, 0x7365656B])
            out[b, h] = C.scrambled_step(ss, b + 1, 0, self.Hkv, h // G, self.q[b, h], self.q_first_pos,
                                         [k[b, h // G] for k in self.k], [v[b, h // G] for v in self.v],
                                         wire_fmt=self.fmt, lo=self.mag[0], hi=self.mag[1], mode=self.mode)
        return out

    def plain(self, pairs=None):
        """Plain unscrambled attention in f64 over the concatenated context."""
        G = self.Hq // self.Hkv
        out = np.zeros_like(self.q)
        pairs = pairs or [(b, h) for b in range(self.B) for h in range(self.Hq)]
        for b, h in pairs:
            kk = np.concatenate([k[b, h // G] for k in self.k])
            vv = np.concatenate([v[b, h // G] for v in self.v])
            out[b, h] = C.shard_attention(self.q[b, h], kk, vv)[0]
        return out
