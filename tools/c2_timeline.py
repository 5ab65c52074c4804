"""Kernel timeline of the C2 decode step (N=1: K1 scramble of Q -> K2 decode -> K3 merge, as
bench.py runs it, CUDA-graph replayed) from the CUDA profiler (CUPTI device timestamps): per
kernel the mean duration, and per step the mean start-to-start offsets K1 -> K2 -> K3 -> next K1.
  S=<splits> python tools/c2_timeline.py"""
import os
import statistics
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops, protocol  # noqa: E402

H, D, L, B = 32, 128, 8192, 16


def main(steps=20):
    dev = torch.device("cuda")
    keys = protocol.DomainKeys(list(range(1, B + 1)), 0, 1, H, D, dev)
    shard = protocol.KVShard(B, H, L, D, dev)
    g = torch.Generator(device=dev).manual_seed(0)
    shard.ship_segment(torch.randn((B, H, L, D), generator=g, device=dev).to(torch.bfloat16),
                       torch.randn((B, H, L, D), generator=g, device=dev).to(torch.bfloat16), keys, 0)
    q = torch.randn((B, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
    S = int(os.environ.get("S", 0)) or capi.default_splits(B, H, 1, L)
    qs = torch.empty_like(q)
    o = torch.empty((S, B, H, 1, D), dtype=torch.float32, device=dev)
    st = torch.empty((S, B, H, 1, 2), dtype=torch.float32, device=dev)
    out = torch.empty((B, H, 1, D), dtype=torch.float32, device=dev)
    srcs = ops.sources_from_splits(o, st, keys.dev, None)

    def step():
        ops.scramble(q, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=qs, key_heads=H)
        ops.partial_attention(qs, shard.k, shard.v, shard.kv_len, n_splits=S, out_o=o, out_stats=st)
        ops.unscramble_merge(srcs, out=out, key_heads=H)

    for _ in range(3):
        step()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(5):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"S={S}; step (events, graph replay): {e0.elapsed_time(e1) * 1e3 / steps:.1f} us")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            gr.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "sda::" in e.name]
    evs.sort(key=lambda e: e.time_range.start)
    kind = lambda n: "K1" if "k1_" in n else ("K2" if "k2_" in n else "K3")  # noqa: E731
    dur = {"K1": [], "K2": [], "K3": []}
    for e in evs:
        dur[kind(e.name)].append(e.time_range.elapsed_us())
    print("kernels:", {k: round(statistics.mean(v), 1) for k, v in dur.items() if v},
          sorted({e.name[:60] for e in evs}))
    seq = [(kind(e.name), e.time_range.start, e.time_range.end) for e in evs]
    offs = {"K1->K2 start": [], "K2->K3 start": [], "K3->K1 start": [], "K1 end->K2 end": [], "K2 end->K3 end": []}
    for i in range(len(seq) - 1):
        a, b = seq[i], seq[i + 1]
        if (a[0], b[0]) == ("K1", "K2"):
            offs["K1->K2 start"].append(b[1] - a[1])
            offs["K1 end->K2 end"].append(b[2] - a[2])
        elif (a[0], b[0]) == ("K2", "K3"):
            offs["K2->K3 start"].append(b[1] - a[1])
            offs["K2 end->K3 end"].append(b[2] - a[2])
        elif (a[0], b[0]) == ("K3", "K1"):
            offs["K3->K1 start"].append(b[1] - a[1])
    print("offsets (us):", {k: round(statistics.median(v), 1) for k, v in offs.items() if v})


if __name__ == "__main__":
    main()
