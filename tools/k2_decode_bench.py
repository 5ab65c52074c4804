"""K2 decode micro-benchmark at BASELINE config 2 (16 requests x 32 heads x 8K keys x d128, bf16):
one launch timed back to back from a CUDA graph, for several split counts; prints TB/s of the
algorithmic bytes (KV + Q' + partials).
  python tools/k2_decode_bench.py [B=<requests> L=<keys>] [splits...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops  # noqa: E402


def main():
    B, H, L, D = 16, 32, 8192, 128
    args = sys.argv[1:]
    if args and args[0].startswith("B="):   # B=<requests> L=<keys> then splits
        B, L = int(args[0][2:]), int(args[1][2:])
        args = args[2:]
    splits = [int(a) for a in args] or [6, 8, 10, 12, 16, 20]
    dev = torch.device("cuda")
    k = torch.randn((B, H, L, D), device=dev).to(torch.bfloat16)
    v = torch.randn((B, H, L, D), device=dev).to(torch.bfloat16)
    q = torch.randn((B, H, 1, D), device=dev).to(torch.bfloat16)
    for S in splits:
        o = torch.empty((S, B, H, 1, D), dtype=torch.float32, device=dev)
        st = torch.empty((S, B, H, 1, 2), dtype=torch.float32, device=dev)
        ops.partial_attention(q, k, v, n_splits=S, out_o=o, out_stats=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                ops.partial_attention(q, k, v, n_splits=S, out_o=o, out_stats=st)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 60
        nbytes = B * H * L * D * 2 * 2 + B * H * D * 2 + S * B * H * (4 * D + 8)
        print(f"K2 decode splits={S:3d}: {us:7.1f} us  {nbytes / us / 1e6:6.3f} TB/s", flush=True)


if __name__ == "__main__":
    main()
