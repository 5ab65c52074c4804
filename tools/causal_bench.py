"""The inquirer's causal local span on the tensor-core prefill kernel (BASELINE cfg3: a 2K-token
span attending its own K/V, 32 heads x d128, bf16), CUDA-event timed per split count.
  python tools/causal_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops  # noqa: E402


def main(H=32, LQ=2048, D=128, reps=20):
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v = (torch.randn((1, H, LQ, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    flops = 2.0 * LQ * (LQ + 1) * H * D
    for S in (1, 2, 3, 4):
        o = torch.empty((S, 1, H, LQ, D), device="cuda")
        st = torch.empty((S, 1, H, LQ, 2), device="cuda")
        for _ in range(3):
            ops.partial_attention_causal(q, k, v, 0, n_splits=S, out_o=o, out_stats=st)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(reps):
                ops.partial_attention_causal(q, k, v, 0, n_splits=S, out_o=o, out_stats=st)
        gr.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        print(f"causal {LQ}x{LQ} x {H} heads, splits {S}: {t * 1e3:.1f} us, {flops / t / 1e9:.0f} TFLOP/s")


if __name__ == "__main__":
    main()
