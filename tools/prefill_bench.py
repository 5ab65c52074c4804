"""Micro-benchmark of the tcgen05 prefill partial attention (K2) at BASELINE config 3 per GPU:
2048-row prefill span x 16K-key scrambled shard x 32 heads x d128 (bf16), CUDA-event timed.
  [HKV=kv_heads] python tools/prefill_bench.py [Lq Lk H splits...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    Lq, Lk, H = (a + [2048, 16384, 32][len(a):])[:3]
    splits = a[3:] or [1, 2, 3, 4, 6, 8]
    D = 128
    dev = torch.device("cuda")
    HKV = int(os.environ.get("HKV", H))   # GQA: kv heads (default = H)
    q = torch.randn((1, H, Lq, D), device=dev).to(torch.bfloat16)
    k = torch.randn((1, HKV, Lk, D), device=dev).to(torch.bfloat16)
    v = torch.randn((1, HKV, Lk, D), device=dev).to(torch.bfloat16)
    flops = 4.0 * Lq * Lk * H * D
    for S in splits:
        ts = []
        for i in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.partial_attention(q, k, v, n_splits=S)
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(f"prefill K2 Lq{Lq} Lk{Lk} H{H} splits={S}: {t * 1e3:8.1f} us  {flops / t / 1e9:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
