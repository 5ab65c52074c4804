"""Micro-benchmark of GQA decode partial attention at BASELINE config 5 per GPU (64 q heads /
8 kv heads x d128, 64K-token scrambled KV shard per request, bf16): grouped tcgen05 kernel vs
the SIMT kernel. CUDA-event timed; KV (8.6 GB at B=32) is far larger than L2.
  python tools/gqa_bench.py [B L [splits...]]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops  # noqa: E402


def main():
    a = [int(x) for x in sys.argv[1:]]
    B, L = (a + [32, 65536][len(a):])[:2]
    sweep = a[2:]   # optional split counts for the tensor-core kernel
    Hq, Hkv, D = 64, 8, 128
    dev = torch.device("cuda")
    q = torch.randn((B, Hq, 1, D), device=dev).to(torch.bfloat16)
    k = torch.empty((B, Hkv, L, D), device=dev, dtype=torch.bfloat16).normal_()
    v = torch.empty((B, Hkv, L, D), device=dev, dtype=torch.bfloat16).normal_()
    nbytes = 2 * k.numel() * 2 + q.numel() * 2
    for impl in (["tc"] * len(sweep) if sweep else ["tc", "simt"]):
        if impl == "simt":
            os.environ["SDA_K2_SIMT"] = "1"
        else:
            os.environ.pop("SDA_K2_SIMT", None)
        S = capi.default_splits(B, Hq, 1, L, kv_heads=Hkv, head_dim=D) if impl == "tc" else \
            capi.default_splits(B, Hq, 1, L)
        if sweep:
            S = sweep.pop(0)
        ts = []
        for i in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.partial_attention(q, k, v, n_splits=S)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        t = float(np.median(ts))
        print(f"GQA decode {impl:4s} B{B} Hq{Hq}/Hkv{Hkv} L{L} splits={S}: {t * 1e3:8.1f} us  "
              f"{nbytes / t / 1e6:7.1f} GB/s  {B / t * 1e3:9.0f} tokens/s")


if __name__ == "__main__":
    main()
