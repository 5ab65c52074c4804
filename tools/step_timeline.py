"""Per-rank device timeline of the multi-GPU decode step (run under torchrun, N >= 2).

A 1-thread %globaltimer kernel (sda_trace_timestamp) is placed between the phases of the step;
STEPS steps are captured unrolled in one CUDA graph (distinct stamp slots) and replayed. Rank 0
prints, per rank, the median duration of every phase and the median offset of each rank's step
start from rank 0's (the globaltimers of the GPUs of one box agree to ~1 us).
  python -m torch.distributed.run --nproc-per-node 4 tools/step_timeline.py [ll|p2p|nccl]"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, protocol  # noqa: E402
from paper_2605_25716_b200 import distributed as sdist  # noqa: E402

H, D, L, B = 32, 128, 8192, 16   # BASELINE cfg2 per GPU
STEPS, REPS = 20, 10


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "ll"
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    Lr, Bt = L // world, B * world
    keys_own = protocol.DomainKeys(list(range(1, Bt + 1)), 0, rank + 1, H, D, dev)
    shard = protocol.KVShard(Bt, H, Lr, D, dev)
    g = torch.Generator(device=dev).manual_seed(rank)
    shard.ship_segment(torch.randn((Bt, H, Lr, D), generator=g, device=dev).to(torch.bfloat16),
                       torch.randn((Bt, H, Lr, D), generator=g, device=dev).to(torch.bfloat16), keys_own, rank * Lr)
    inq = [protocol.DomainKeys(list(range(rank * B + 1, rank * B + B + 1)), 0, d + 1, H, D, dev) for d in range(world)]
    bufs = sdist.StepBuffers.allocate(world, B, H, 1, D, torch.bfloat16, dev)
    comp = sdist.gpu_rank_compute(inq, shard, kv_heads=H)
    q = torch.randn((B, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
    out = torch.empty((B, H, 1, D), dtype=torch.float32, device=dev)
    stamps = torch.zeros((STEPS, 16), dtype=torch.int64, device=dev)
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    qa, ret = bufs.q_recv.view(Bt, H, 1, D), bufs.ret_send.view(Bt, -1)

    if mode == "ll":
        lld = sdist.LLDecode(B, H, D, inq, shard, kv_heads=H)
        names = ["K1 (+Q' out)", "K2 (+Q' in, records out)", "K3 (+records in)"]
        fns = [lambda: lld.scramble_q(q), lld.serve, lambda: lld.finish(out)]
    elif mode == "p2p":
        ex = sdist.PeerExchange(bufs)
        names = ["epoch", "K1", "push Q", "wait Q", "K2+fold", "push ret", "wait ret", "K3"]
        fns = [ex.begin_step, lambda: comp.scramble_q_all(q, bufs.q_send), lambda: ex._push(ex.q_args, 0),
               lambda: ex._wait(0), lambda: comp.serve(qa, ret, bufs.dims), lambda: ex._push(ex.r_args, world),
               lambda: ex._wait(world), lambda: comp.finish(bufs.ret_recv, out, bufs.dims)]
    else:
        names = ["K1", "a2a Q", "K2+fold", "a2a ret", "K3"]
        fns = [lambda: comp.scramble_q_all(q, bufs.q_send), lambda: dist.all_to_all_single(bufs.q_recv, bufs.q_send),
               lambda: comp.serve(qa, ret, bufs.dims), lambda: dist.all_to_all_single(bufs.ret_recv, bufs.ret_send),
               lambda: comp.finish(bufs.ret_recv, out, bufs.dims)]

    def one_step(i):
        capi.LIB.sda_trace_timestamp(st(), stamps[i].data_ptr())
        for j, fn in enumerate(fns):
            fn()
            capi.LIB.sda_trace_timestamp(st(), stamps[i].data_ptr() + 8 * (j + 1))

    for i in range(3):
        one_step(i)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(STEPS):
            one_step(i)
    dist.barrier(device_ids=[local])
    rows = []
    for _ in range(REPS):
        graph.replay()
        torch.cuda.synchronize()
        rows.append(stamps.clone())
    allst = torch.stack(rows).view(-1, 16)[:, :len(fns) + 1].contiguous()         # [REPS*STEPS, phases+1]
    gathered = [torch.empty_like(allst) for _ in range(world)]
    dist.all_gather(gathered, allst)
    if rank == 0:
        base = gathered[0][:, 0]
        print(f"mode {mode}, world {world}: median us per phase (and step start offset vs rank 0)")
        for r in range(world):
            t = gathered[r].double()
            dur = (t[:, 1:] - t[:, :-1]) / 1e3
            med = dur.median(0).values.tolist()
            tot = ((t[:, -1] - t[:, 0]) / 1e3).median().item()
            period = ((t[1:, 0] - t[:-1, 0]) / 1e3).median().item()
            off = ((t[:, 0] - base.double()) / 1e3).median().item()
            print(f"  rank {r}: " + ", ".join(f"{n} {m:.1f}" for n, m in zip(names, med)) +
                  f" | step {tot:.1f}, period {period:.1f}, start offset {off:+.1f}", flush=True)
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    os._exit(0)


if __name__ == "__main__":
    main()
