"""The scrambled-attention data path of the reference protocol, one compute domain at a time.

Maps the reference's message handlers onto device calls (all compute in libsdattn_b200.so):

  ship_segment_kv   (protocol.cpp:987-1016)  -> KVShard.ship_segment: K1 K' = K phi_kq^{-T},
                                               V' = V phi_v, rows gathered by span_perm(1, ...),
                                               written straight into the resident cache
  on_scr_kv         (protocol.cpp:1021-1040) -> the cache *is* the store (no frame decode)
  span_send_layer   (protocol.cpp:876-899)   -> DomainKeys.scramble_q: K1 Q' = Q phi_kq, p_q
  try_serve_q       (protocol.cpp:1053-1104) -> KVShard.serve: K2 over the resident shard
  span_finish_layer (protocol.cpp:921-949)   -> finish(): K3 dec_output + merge_shards

Key material: one DomainKeys per (requests, layer, domain). The compute node of a domain only
ever holds KVShard (scrambled tensors) -- it never sees DomainKeys (role rule,
protocol.cpp:215-216).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch

from . import capi, ops


class DomainKeys:
    """Θ for a batch of requests on one (layer, domain): host key sets + packed device image.

    requests are (master_seed, request_id) pairs; shared seed per request is
    derive_seed(master, {request_id, 0x7365656B}) (protocol.cpp:143-145). For GQA the feature
    scramblers are per kv head (the reference rule with head tag = kv head).
    """

    def __init__(self, request_ids: Sequence[int], layer: int, domain: int, kv_heads: int, head_dim: int,
                 device, master_seed: int = 1, mag_lo: float = 0.125, mag_hi: float = 8.0,
                 mode: int = capi.MODE_S1_AND_S2, shared_seeds: Optional[Sequence[int]] = None,
                 fp64: bool = False):
        """fp64: upload the FP64-mode key image (for f64 activations / shards) instead of the f32 one."""
        self.request_ids = list(request_ids)
        self.layer, self.domain = layer, domain
        self.kv_heads, self.head_dim = kv_heads, head_dim
        self.device = torch.device(device)
        seeds = shared_seeds if shared_seeds is not None else [capi.shared_seed(master_seed, r) for r in request_ids]
        self.host = [capi.negotiate_keyset(s, r, layer, domain, kv_heads, head_dim, mag_lo, mag_hi, mode)
                     for s, r in zip(seeds, self.request_ids)]
        self.fp64 = fp64
        self.dev = ops.upload_keys([ks.pack_f64() if fp64 else ks.pack() for ks in self.host], self.device)

    @property
    def batch(self) -> int:
        return len(self.request_ids)

    def span_perms(self, tag: int, first_pos: int, length: int):
        """(forward, inverse) device int32 [B, length] for span_perm(tag, first_pos, length)."""
        fwd = [ks.span_perm(tag, first_pos, length) for ks in self.host]
        inv = [capi.invert_permutation(p) for p in fwd]
        return ops.upload_perms(fwd, self.device), ops.upload_perms(inv, self.device)

    def scramble_q(self, q: torch.Tensor, q_first_pos: int, out_dtype=None, stream=None):
        """Q' = gather_rows(Q phi_kq, p_q) for every request. Returns (q', p_q^{-1} or None)."""
        rows = q.shape[2]
        if rows == 1:  # span_perm over one row is the identity
            return ops.scramble(q, self.dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out_dtype=out_dtype,
                                key_heads=self.kv_heads, stream=stream), None
        p, pinv = self.span_perms(0, q_first_pos, rows)
        return ops.scramble(q, self.dev, capi.PHI_FORWARD, capi.KEYS_KQ, p, out_dtype=out_dtype,
                            key_heads=self.kv_heads, stream=stream), pinv


class KVShard:
    """A compute node's resident scrambled KV for one domain: k, v [B, Hkv, cap, d]."""

    def __init__(self, batch: int, kv_heads: int, capacity: int, head_dim: int, device,
                 dtype: torch.dtype = torch.bfloat16):
        self.k = torch.zeros((batch, kv_heads, capacity, head_dim), dtype=dtype, device=device)
        self.v = torch.zeros_like(self.k)
        self.kv_len = torch.zeros(batch, dtype=torch.int32, device=device)
        self.rows = 0

    @property
    def capacity(self) -> int:
        return self.k.shape[2]

    def ship_segment(self, k_plain: torch.Tensor, v_plain: torch.Tensor, keys: DomainKeys, first_pos: int,
                     stream=None) -> None:
        """Context owner side of ship_segment_kv: scramble + permute one segment [B, Hkv, L, d]
        into the cache rows [self.rows, self.rows + L) (each segment is shuffled within itself,
        span_perm(1, first_pos, L), scrambler.cpp:99-103)."""
        L = k_plain.shape[2]
        if self.rows + L > self.capacity:
            raise ValueError("KV shard capacity exceeded")
        p, _ = keys.span_perms(1, first_pos, L)
        # K' = K phi_KQ^{-T} and V' = V phi_V, both permuted by p, in one K1 launch
        ops.scramble_batch([ops.scramble_job(k_plain, keys.dev, capi.PHI_INV_T, capi.KEYS_KQ, p, out=self.k,
                                             out_row_offset=self.rows, key_heads=keys.kv_heads),
                            ops.scramble_job(v_plain, keys.dev, capi.PHI_FORWARD, capi.KEYS_V, p, out=self.v,
                                             out_row_offset=self.rows, key_heads=keys.kv_heads)],
                           k_plain.shape[3], stream=stream)
        self.rows += L
        self.kv_len.fill_(self.rows)

    def serve(self, q_scr: torch.Tensor, n_splits: Optional[int] = None, stream=None):
        """try_serve_q: keyless partial attention over the whole resident shard."""
        return ops.partial_attention(q_scr, self.k, self.v, self.kv_len, n_splits=n_splits, stream=stream)


def finish(partials: Sequence, out_dtype=torch.float32, kv_heads: Optional[int] = None,
           local: Sequence = (), err_flag: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """span_finish_layer: partials = [(o [S,...], stats [S,...], DomainKeys, pq_inv)] per domain;
    local = [(o, stats)] plaintext shards of the inquirer (no unscramble)."""
    sources: List[ops.MergeSource] = []
    for o, st, keys, pq_inv in partials:
        sources += ops.sources_from_splits(o, st, keys.dev, pq_inv)
    for o, st in local:
        sources += ops.sources_from_splits(o, st, None, None)
    return ops.unscramble_merge(sources, out_dtype=out_dtype, key_heads=kv_heads, err_flag=err_flag, stream=stream)


def scrambled_attention(q: torch.Tensor, domains: Sequence, q_first_pos: int, n_splits: Optional[int] = None,
                        out_dtype=torch.float32, stream=None) -> torch.Tensor:
    """One scrambled-attention layer step for a batch: for every (DomainKeys, KVShard) pair,
    K1 scramble Q -> K2 on the shard -> K3 merge all domains. Single-device form (the
    multi-GPU form moves Q' and the partials over NCCL, see distributed.py)."""
    partials = []
    kv_heads = None
    for keys, shard in domains:
        q_s, pinv = keys.scramble_q(q, q_first_pos, out_dtype=shard.k.dtype, stream=stream)
        o, st = shard.serve(q_s, n_splits=n_splits, stream=stream)
        partials.append((o, st, keys, pinv))
        kv_heads = keys.kv_heads
    return finish(partials, out_dtype=out_dtype, kv_heads=kv_heads, stream=stream)


def as_numpy_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to(torch.float64).cpu().numpy()
