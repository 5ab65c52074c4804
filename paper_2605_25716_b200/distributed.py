"""Multi-GPU form of the scrambled decode step: one process per GPU, one compute domain per GPU.

The reference moves SCR_Q frames inquirer -> compute node and SCR_SHARD frames back
(protocol.cpp:892-896, :1097-1102) over its simulated network. Here every rank is both
  * the compute node of domain `rank + 1` (it holds that domain's scrambled KV shard for all
    requests and runs K2 on whatever Q' arrives), and
  * the inquirer for its own slice of requests (it scrambles their Q once per destination
    domain, K1, and merges + unscrambles the returning partials, K3).
One layer step is therefore: K1 x world -> all_to_all(Q') -> K2 -> split fold -> all_to_all(O',
stats) -> K3. It is not an all-reduce: each domain's partial must be unscrambled with that
domain's phi_V^{-1}, which only the key holder has.

The exchange is plain torch.distributed all_to_all_single (NCCL over NVLink on the GPU box,
gloo in the CPU tests); the per-rank compute is pluggable so the routing logic can be tested
on CPU with the oracle standing in for the kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist


@dataclass
class StepBuffers:
    """Preallocated exchange buffers for one rank (world W, B_p requests per inquirer)."""
    q_send: torch.Tensor    # [W, B_p, Hq, Lq, d]   Q' for each destination domain
    q_recv: torch.Tensor    # [W, B_p, Hq, Lq, d]   Q' from each inquirer = [W*B_p, ...] for K2
    o_fold: torch.Tensor    # [W, B_p, Hq, Lq, d]   this domain's partial per inquirer (f32)
    st_fold: torch.Tensor   # [W, B_p, Hq, Lq, 2]
    o_back: torch.Tensor    # [W, B_p, Hq, Lq, d]   partial of every domain for my requests
    st_back: torch.Tensor   # [W, B_p, Hq, Lq, 2]

    @staticmethod
    def allocate(world: int, b_per: int, q_heads: int, q_rows: int, d: int, q_dtype, device) -> "StepBuffers":
        shp = (world, b_per, q_heads, q_rows, d)
        f32 = dict(dtype=torch.float32, device=device)
        return StepBuffers(torch.empty(shp, dtype=q_dtype, device=device),
                           torch.empty(shp, dtype=q_dtype, device=device),
                           torch.empty(shp, **f32), torch.empty(shp[:-1] + (2,), **f32),
                           torch.empty(shp, **f32), torch.empty(shp[:-1] + (2,), **f32))


@dataclass
class RankCompute:
    """The per-rank compute of one step (GPU: the K1/K2/K3 calls of ops.py)."""
    scramble_q: Callable[[torch.Tensor, int, torch.Tensor], None]          # (q, dst_domain, out)
    serve: Callable[[torch.Tensor, torch.Tensor, torch.Tensor], None]       # (q_all, o_out, st_out) K2 + fold
    finish: Callable[[torch.Tensor, torch.Tensor, torch.Tensor], None]      # (o_back, st_back, out) K3


def scrambled_decode_step(q: torch.Tensor, compute: RankCompute, bufs: StepBuffers, out: torch.Tensor,
                          group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """One layer step for this rank's requests q [B_p, Hq, Lq, d]; returns out [B_p, Hq, Lq, d]."""
    world = bufs.q_send.shape[0]
    for dom in range(world):                                     # span_send_layer, per domain
        compute.scramble_q(q, dom, bufs.q_send[dom])
    if world > 1:
        dist.all_to_all_single(bufs.q_recv, bufs.q_send, group=group)   # SCR_Q
        q_all = bufs.q_recv
    else:
        q_all = bufs.q_send
    b_tot = q_all.shape[0] * q_all.shape[1]
    compute.serve(q_all.view((b_tot,) + tuple(q_all.shape[2:])),     # try_serve_q on my shard
                  bufs.o_fold.view((b_tot,) + tuple(bufs.o_fold.shape[2:])),
                  bufs.st_fold.view((b_tot,) + tuple(bufs.st_fold.shape[2:])))
    if world > 1:
        dist.all_to_all_single(bufs.o_back, bufs.o_fold, group=group)    # SCR_SHARD (O')
        dist.all_to_all_single(bufs.st_back, bufs.st_fold, group=group)  # SCR_SHARD (stats)
        o_back, st_back = bufs.o_back, bufs.st_back
    else:
        o_back, st_back = bufs.o_fold, bufs.st_fold
    compute.finish(o_back, st_back, out)                          # span_finish_layer
    return out


def gpu_rank_compute(inquirer_keys: Sequence, shard, n_splits: Optional[int] = None,
                     kv_heads: Optional[int] = None) -> RankCompute:
    """RankCompute backed by libsdattn_b200.so. inquirer_keys[dom] = DomainKeys of my requests on
    domain dom + 1; shard = this rank's protocol.KVShard (all requests' rows of my domain)."""
    from . import capi, ops

    state = {}

    def scramble_q(q, dom, out):
        ops.scramble(q, inquirer_keys[dom].dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=out,
                     key_heads=kv_heads or inquirer_keys[dom].kv_heads)

    def serve(q_all, o_out, st_out):
        B, Hq, Lq, d = q_all.shape
        S = n_splits or capi.default_splits(B, Hq, Lq, shard.capacity)
        key = (S, B, Hq, Lq, d)
        if state.get("key") != key:
            state["key"] = key
            state["o"] = torch.empty((S, B, Hq, Lq, d), dtype=torch.float32, device=q_all.device)
            state["st"] = torch.empty((S, B, Hq, Lq, 2), dtype=torch.float32, device=q_all.device)
        ops.partial_attention(q_all, shard.k, shard.v, shard.kv_len, n_splits=S, out_o=state["o"],
                              out_stats=state["st"])
        # fold the splits of this domain in scrambled space (plain merge, no keys): one O' and one
        # (row_max, exp_sum) per request row, exactly what SCR_SHARD carries
        ops.unscramble_merge(ops.sources_from_splits(state["o"], state["st"]), out=o_out, out_stats=st_out)

    def finish(o_back, st_back, out):
        srcs = [ops.MergeSource(o_back[dom], st_back[dom], inquirer_keys[dom].dev, None)
                for dom in range(o_back.shape[0])]
        ops.unscramble_merge(srcs, out=out, key_heads=kv_heads or inquirer_keys[0].kv_heads)

    return RankCompute(scramble_q, serve, finish)
