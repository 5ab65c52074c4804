"""Per-phase device time of the decode step on one GPU (CUDA events between phases, eager):
the N=1 path (K1 -> K2 -> K3) and the multi-GPU path at world 1 (K1 -> K2 -> split fold into
packed records -> K3), cfg2 sizes.  python tools/step_breakdown.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops, protocol  # noqa: E402
from paper_2605_25716_b200 import distributed as sdist  # noqa: E402

H, D, L, B = 32, 128, 8192, 16


def timed(phases, n=50):
    st = torch.cuda.current_stream()
    acc = {name: [] for name, _ in phases}
    for _ in range(n):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(phases) + 1)]
        evs[0].record(st)
        for i, (name, fn) in enumerate(phases):
            fn()
            evs[i + 1].record(st)
        torch.cuda.synchronize()
        for i, (name, _) in enumerate(phases):
            acc[name].append(evs[i].elapsed_time(evs[i + 1]) * 1e3)
    return {k: statistics.median(v) for k, v in acc.items()}


def main():
    dev = torch.device("cuda")
    keys = protocol.DomainKeys(list(range(1, B + 1)), 0, 1, H, D, dev)
    shard = protocol.KVShard(B, H, L, D, dev)
    g = torch.Generator(device=dev).manual_seed(0)
    shard.ship_segment(torch.randn((B, H, L, D), generator=g, device=dev).to(torch.bfloat16),
                       torch.randn((B, H, L, D), generator=g, device=dev).to(torch.bfloat16), keys, 0)
    q = torch.randn((B, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
    S = capi.default_splits(B, H, 1, L)
    qs = torch.empty_like(q)
    o = torch.empty((S, B, H, 1, D), dtype=torch.float32, device=dev)
    st = torch.empty((S, B, H, 1, 2), dtype=torch.float32, device=dev)
    out = torch.empty((B, H, 1, D), dtype=torch.float32, device=dev)
    srcs = ops.sources_from_splits(o, st, keys.dev, None)
    for _ in range(3):
        ops.scramble(q, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=qs, key_heads=H)
    r1 = timed([("K1 Q", lambda: ops.scramble(q, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=qs, key_heads=H)),
                ("K2", lambda: ops.partial_attention(qs, shard.k, shard.v, shard.kv_len, n_splits=S, out_o=o, out_stats=st)),
                ("K3 merge+unscramble", lambda: ops.unscramble_merge(srcs, out=out, key_heads=H))])
    print("N=1 path:", {k: round(v, 1) for k, v in r1.items()}, "total us", round(sum(r1.values()), 1))
    bufs = sdist.StepBuffers.allocate(1, B, H, 1, D, torch.bfloat16, dev)
    comp = sdist.gpu_rank_compute([keys], shard, n_splits=S, kv_heads=H)
    qa = bufs.q_send.view(B, H, 1, D)
    ret = bufs.ret_send.view(B, -1)
    r2 = timed([("K1 Q (all domains)", lambda: comp.scramble_q_all(q, bufs.q_send)),
                ("K2 + split fold", lambda: comp.serve(qa, ret, bufs.dims)),
                ("K3 from packed records", lambda: comp.finish(bufs.ret_send, out, bufs.dims))])
    print("multi-GPU path (world 1):", {k: round(v, 1) for k, v in r2.items()}, "total us", round(sum(r2.values()), 1))


def multi():
    """Under torchrun: per-phase device time of the peer-exchange step on every rank."""
    import torch.distributed as dist
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    Lr = L // world
    Bt = B * world
    keys_own = protocol.DomainKeys(list(range(1, Bt + 1)), 0, rank + 1, H, D, dev)
    shard = protocol.KVShard(Bt, H, Lr, D, dev)
    g = torch.Generator(device=dev).manual_seed(rank)
    shard.ship_segment(torch.randn((Bt, H, Lr, D), generator=g, device=dev).to(torch.bfloat16),
                       torch.randn((Bt, H, Lr, D), generator=g, device=dev).to(torch.bfloat16), keys_own, rank * Lr)
    inq = [protocol.DomainKeys(list(range(rank * B + 1, rank * B + B + 1)), 0, d + 1, H, D, dev) for d in range(world)]
    bufs = sdist.StepBuffers.allocate(world, B, H, 1, D, torch.bfloat16, dev)
    comp = sdist.gpu_rank_compute(inq, shard, kv_heads=H)
    ex = sdist.PeerExchange(bufs)
    q = torch.randn((B, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
    out = torch.empty((B, H, 1, D), dtype=torch.float32, device=dev)
    qa = bufs.q_recv.view(Bt, H, 1, D)
    ret = bufs.ret_send.view(Bt, -1)
    phases = [("epoch", ex.begin_step), ("K1", lambda: comp.scramble_q_all(q, bufs.q_send)),
              ("push Q", lambda: ex._push(ex.q_args, 0)), ("wait Q", lambda: ex._wait(0)),
              ("K2+fold", lambda: comp.serve(qa, ret, bufs.dims)), ("push ret", lambda: ex._push(ex.r_args, world)),
              ("wait ret", lambda: ex._wait(world)), ("K3", lambda: comp.finish(bufs.ret_recv, out, bufs.dims))]
    for _ in range(5):
        for _, fn in phases:
            fn()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    r = timed(phases, 50)
    print(f"rank {rank}:", {k: round(v, 1) for k, v in r.items()}, "sum", round(sum(r.values()), 1), flush=True)
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    os._exit(0)


if __name__ == "__main__" and "RANK" in os.environ:
    multi()
elif __name__ == "__main__":
    main()
