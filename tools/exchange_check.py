"""Multi-GPU check of the peer-memory exchange (run under torchrun, N >= 2): the same decode
steps through NCCL all-to-all and through exchange.cu must give bit-identical outputs, over many
steps (epoch logic) and inside a CUDA graph; the first step of every form is also checked against
the oracle's W-node composition (C.scrambled_step) on the oracle's seeded inputs. Prints one line per rank; exits non-zero on mismatch.
  python -m torch.distributed.run --nproc-per-node 2 tools/exchange_check.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops, protocol  # noqa: E402
from paper_2605_25716_b200 import distributed as sdist  # noqa: E402
from tests.gpu_helpers import Case, max_abs_rel, rel_fro  # noqa: E402


def dev_(x, device):
    return torch.from_numpy(x).to(device).to(torch.bfloat16)


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    H, D, L, BP = 8, 128, 1024, 4
    B = BP * world
    # the oracle's seeded inputs (identical on every rank): rank r holds domain r + 1's shard
    case = Case(B=B, Hq=H, Hkv=H, d=D, lk=L, n_nodes=world, lq=1, dtype=torch.bfloat16, seed=41)
    keys_own = protocol.DomainKeys(list(range(1, B + 1)), 0, rank + 1, H, D, dev)
    shard = protocol.KVShard(B, H, L, D, dev)
    g = torch.Generator(device=dev).manual_seed(rank)
    shard.ship_segment(dev_(case.k[rank], dev), dev_(case.v[rank], dev), keys_own, first_pos=rank * L)
    inq = [protocol.DomainKeys(list(range(rank * BP + 1, rank * BP + BP + 1)), 0, d + 1, H, D, dev) for d in range(world)]
    bufs = sdist.StepBuffers.allocate(world, BP, H, 1, D, torch.bfloat16, dev)
    comp = sdist.gpu_rank_compute(inq, shard, kv_heads=H)
    exch = sdist.PeerExchange(bufs)
    fused = sdist.LLDecode(BP, H, D, inq, shard, kv_heads=H)
    out_n = torch.empty((BP, H, 1, D), dtype=torch.float32, device=dev)
    out_p = torch.empty_like(out_n)
    out_f = torch.empty_like(out_n)
    ok = True
    worst_f = 0.0
    # step 0 against the oracle's W-node composition (C.scrambled_step), every form
    q0 = dev_(case.q[rank * BP:(rank + 1) * BP], dev)
    sdist.scrambled_decode_step(q0, comp, bufs, out_n)
    sdist.scrambled_decode_step(q0, comp, bufs, out_p, exchange=exch)
    fused.step(q0, out_f)
    torch.cuda.synchronize()
    pairs = [(rank * BP + i, h) for i in range(BP) for h in (0, 3, H - 1)]
    ref = case.oracle(pairs)
    worst_o = 0.0
    for o in (out_n, out_p, out_f):
        got = o.double().cpu().numpy()
        for b, h in pairs:
            worst_o = max(worst_o, max_abs_rel(got[b - rank * BP, h], ref[b, h]), rel_fro(got[b - rank * BP, h], ref[b, h]))
    ok_o = worst_o < 2e-2
    for it in range(20):
        q = torch.randn((BP, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
        sdist.scrambled_decode_step(q, comp, bufs, out_n)
        sdist.scrambled_decode_step(q, comp, bufs, out_p, exchange=exch)
        fused.step(q, out_f)
        torch.cuda.synchronize()
        ok &= bool(torch.equal(out_n, out_p)) and bool(torch.isfinite(out_p).all())
        # the LL path merges the K2 splits inside K3 (one merge over domains x splits) instead of
        # folding them per domain first: same math, different rounding order
        worst_f = max(worst_f, float((out_f - out_n).abs().max() / out_n.abs().max()))
    # inside a CUDA graph, replayed
    q_static = torch.randn((BP, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        sdist.scrambled_decode_step(q_static, comp, bufs, out_p, exchange=exch)
    graph_f = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph_f):
        fused.step(q_static, out_f)
    for it in range(10):
        q_static.copy_(torch.randn((BP, H, 1, D), generator=g, device=dev).to(torch.bfloat16))
        graph.replay()
        graph_f.replay()
        torch.cuda.synchronize()
        sdist.scrambled_decode_step(q_static, comp, bufs, out_n)
        torch.cuda.synchronize()
        ok &= bool(torch.equal(out_n, out_p))
        worst_f = max(worst_f, float((out_f - out_n).abs().max() / out_n.abs().max()))
    ok_f = worst_f < 1e-5
    # prefill spans (256 rows): the return path written by K2 itself into the inquirers' slots
    # (sda_partial_attention_remote, one split) against the NCCL form with the same single split
    # (different split counts round P to bf16 against different bases: ~1e-3 apart)
    LQ, BQ = 256, 1
    inq_p = [protocol.DomainKeys(list(range(rank * BQ + 1, rank * BQ + BQ + 1)), 0, d + 1, H, D, dev) for d in range(world)]
    keys_p = protocol.DomainKeys(list(range(1, world * BQ + 1)), 0, rank + 1, H, D, dev)
    shard_p = protocol.KVShard(world * BQ, H, L, D, dev)
    shard_p.ship_segment(torch.randn((world * BQ, H, L, D), generator=g, device=dev).to(torch.bfloat16),
                         torch.randn((world * BQ, H, L, D), generator=g, device=dev).to(torch.bfloat16), keys_p,
                         first_pos=rank * L)
    comp_p = sdist.gpu_rank_compute(inq_p, shard_p, n_splits=1, kv_heads=H, q_first_pos=world * L)
    bufs_n = sdist.StepBuffers.allocate(world, BQ, H, LQ, D, torch.bfloat16, dev)
    bufs_r = sdist.StepBuffers.allocate(world, BQ, H, LQ, D, torch.bfloat16, dev)
    exch_r = sdist.PeerExchange(bufs_r)
    pn = torch.empty((BQ, H, LQ, D), dtype=torch.float32, device=dev)
    pr = torch.empty_like(pn)
    worst_p = 0.0
    for it in range(5):
        q = torch.randn((BQ, H, LQ, D), generator=g, device=dev).to(torch.bfloat16)
        sdist.scrambled_decode_step(q, comp_p, bufs_n, pn)
        sdist.scrambled_decode_step(q, comp_p, bufs_r, pr, exchange=exch_r)
        torch.cuda.synchronize()
        worst_p = max(worst_p, float((pr - pn).abs().max() / pn.abs().max()))
    ok_p = worst_p < 1e-5
    ok &= ok_p
    print(f"rank {rank}: peer exchange == NCCL over 30 steps (eager + graph): {ok}; "
          f"LL exchange max rel diff {worst_f:.2e}; prefill remote records max rel diff {worst_p:.2e}; "
          f"NCCL / push / LL vs oracle {worst_o:.2e} ({'ok' if ok_f and ok_p and ok_o else 'FAIL'})", flush=True)
    ok &= ok_f and ok_o
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    sys.stdout.flush()
    os._exit(0 if ok else 1)


if __name__ == "__main__":
    main()
