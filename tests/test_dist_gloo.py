"""World-size-2 (and 3) CPU test of the multi-GPU routing in distributed.py over gloo.

Each rank is a compute domain holding its scrambled shard of every request's context and the
inquirer for its own requests; the oracle (reference algorithm in C) stands in for the kernels.
The merged result of every request must equal plain attention over its whole context."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_25716_b200.distributed import RankCompute, StepBuffers, record_views, scrambled_decode_step

H, D, LK, BP = 2, 16, 24, 2   # heads, head dim, rows per domain per request, requests per inquirer


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plain_inputs(world):
    from oracle import C
    B = BP * world
    q = C.gaussian(1, B * H * D).reshape(B, H, 1, D)
    k = C.gaussian(2, world * B * H * LK * D).reshape(world, B, H, LK, D)
    v = C.gaussian(3, world * B * H * LK * D).reshape(world, B, H, LK, D)
    return q, k, v


def _keys(b, dom):
    from oracle import C
    ss = C.derive_seed(1, [b + 1, 0x7365656B])
    return C.negotiate_keyset(ss, b + 1, 0, dom + 1, H, D)


def _sc(ks, h, which):
    p = "kq" if which == 0 else "v"
    return ks[p + "_s1"][h], ks[p + "_p1"][h], ks[p + "_p2"][h], ks[p + "_s2"][h]


def _oracle_compute(rank, world, k, v):
    from oracle import C
    B = BP * world
    # the context owner ships this domain's scrambled + permuted shard (protocol.cpp:987-1016)
    kp, vp = np.zeros((B, H, LK, D)), np.zeros((B, H, LK, D))
    for b in range(B):
        ks = _keys(b, rank)
        p = C.span_perm(ks["token_perm_seed"], 1, rank * LK, LK)
        for h in range(H):
            kp[b, h] = C.apply_phi(k[rank, b, h], *_sc(ks, h, 0), 1)[p]
            vp[b, h] = C.apply_phi(v[rank, b, h], *_sc(ks, h, 1), 0)[p]

    def scramble_q(q, dom, out):
        for i in range(BP):
            ks = _keys(rank * BP + i, dom)
            for h in range(H):
                out[i, h] = torch.from_numpy(C.apply_phi(q[i, h].numpy(), *_sc(ks, h, 0), 0))

    def serve(q_all, ret, dims):
        o_out, st_out = record_views(ret, dims)
        for b in range(B):
            for h in range(H):
                o, m, s = C.shard_attention(q_all[b, h].numpy(), kp[b, h], vp[b, h])
                o_out[b, h] = torch.from_numpy(o)
                st_out[b, h, :, 0] = torch.from_numpy(m)
                st_out[b, h, :, 1] = torch.from_numpy(s)

    def finish(back, out, dims):
        o_back, st_back = record_views(back, dims)
        for i in range(BP):
            for h in range(H):
                outs, ms, ss = [], [], []
                for dom in range(world):
                    ks = _keys(rank * BP + i, dom)
                    outs.append(C.apply_phi(o_back[dom, i, h].numpy(), *_sc(ks, h, 1), 2))
                    ms.append(st_back[dom, i, h, :, 0].numpy())
                    ss.append(st_back[dom, i, h, :, 1].numpy())
                out[i, h] = torch.from_numpy(C.merge_shards(outs, ms, ss))

    return RankCompute(scramble_q, serve, finish)


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import C
        q, k, v = _plain_inputs(world)
        comp = _oracle_compute(rank, world, k, v)
        f64 = dict(dtype=torch.float64)
        shp = (world, BP, H, 1, D)
        rec = H * 1 * (D + 2)
        bufs = StepBuffers(torch.empty(shp, **f64), torch.empty(shp, **f64), torch.empty((world, BP, rec), **f64),
                           torch.empty((world, BP, rec), **f64), (H, 1, D))
        out = torch.empty((BP, H, 1, D), **f64)
        mine = torch.from_numpy(q[rank * BP:(rank + 1) * BP].copy())
        scrambled_decode_step(mine, comp, bufs, out)
        worst = 0.0
        for i in range(BP):
            b = rank * BP + i
            for h in range(H):
                kk = np.concatenate([k[dom, b, h] for dom in range(world)])
                vv = np.concatenate([v[dom, b, h] for dom in range(world)])
                plain = C.shard_attention(q[b, h], kk, vv)[0]
                worst = max(worst, float(np.abs(out[i, h].numpy() - plain).max()))
        ret[rank] = worst
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_scrambled_decode_step_gloo(world):
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.start_processes(_worker, args=(world, port, ret), nprocs=world, join=True, start_method="spawn")
    assert len(ret) == world
    for r in range(world):
        assert ret[r] < 1e-8, (r, ret[r])


@pytest.mark.parametrize("world", [2, 4])
def test_local_world_decode_step_cpu(world):
    """distributed.LocalWorld drives W ranks' decode_step_phases in lockstep in one process (the
    NCCL all-to-alls as slot copies): with the oracle standing in for the kernels, every rank's
    requests must equal plain attention over their whole context -- the same routing the gloo
    test checks across processes, and the driver the GPU emulation tests use."""
    from oracle import C
    from paper_2605_25716_b200.distributed import LocalWorld
    q, k, v = _plain_inputs(world)
    comps = [_oracle_compute(r, world, k, v) for r in range(world)]
    f64 = dict(dtype=torch.float64)
    shp = (world, BP, H, 1, D)
    rec = H * 1 * (D + 2)
    bufs = [StepBuffers(torch.empty(shp, **f64), torch.empty(shp, **f64), torch.empty((world, BP, rec), **f64),
                        torch.empty((world, BP, rec), **f64), (H, 1, D)) for _ in range(world)]
    outs = [torch.empty((BP, H, 1, D), **f64) for _ in range(world)]
    qs = [torch.from_numpy(q[r * BP:(r + 1) * BP].copy()) for r in range(world)]
    LocalWorld.decode_step(qs, comps, bufs, outs)
    for r in range(world):
        for i in range(BP):
            b = r * BP + i
            for h in range(H):
                kk = np.concatenate([k[dom, b, h] for dom in range(world)])
                vv = np.concatenate([v[dom, b, h] for dom in range(world)])
                plain = C.shard_attention(q[b, h], kk, vv)[0]
                assert np.abs(outs[r][i, h].numpy() - plain).max() < 1e-8, (r, i, h)
