"""Library comparison for the prefill K2 at BASELINE config 3 per GPU (2048 q rows x 16384 keys x
32 heads x d128, bf16, no mask): this repo's tcgen05 K2 (stream-K, one split) against the
Blackwell flash-attention kernels in the image -- the CuTe-DSL FA4 forward vendored in vllm
(vllm.vllm_flash_attn.cute, JIT-compiled on first call) and cuDNN through torch SDPA. Library
code, timed only as a yardstick for the K2 roofline discussion in DESIGN.md; CUDA-event timed,
median of 20 after 5 warm-ups; K and V are 2 x 128 MB, larger than the 126 MB L2.
  [ONLY=ours|fa4|cudnn|fa2] python tools/fa_compare.py [Lq Lk H]   (ONLY: one implementation, e.g. under ncu)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops  # noqa: E402


def timeit(fn, n=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts))


def main():
    a = [int(x) for x in sys.argv[1:]]
    Lq, Lk, H = (a + [2048, 16384, 32][len(a):])[:3]
    D = 128
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn((1, H, Lq, D), generator=g, device=dev).to(torch.bfloat16)
    k = torch.randn((1, H, Lk, D), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((1, H, Lk, D), generator=g, device=dev).to(torch.bfloat16)
    flops = 4.0 * Lq * Lk * H * D
    res = {}
    only = os.environ.get("ONLY")
    want = lambda n: only is None or only == n  # noqa: E731
    o_ours = torch.empty((1, 1, H, Lq, D), dtype=torch.float32, device=dev)
    st = torch.empty((1, 1, H, Lq, 2), dtype=torch.float32, device=dev)
    res["ours k2_prefill_tc (f32 O + stats)"] = timeit(n=20 if want("ours") else 1, warm=5 if want("ours") else 0, fn=
        lambda: ops.partial_attention(q, k, v, n_splits=1, out_o=o_ours, out_stats=st))
    # reference output for the checks below (f32 O of the same inputs)
    ref = o_ours[0, 0].float()

    qb, kb, vb = (x.transpose(1, 2).contiguous() for x in (q, k, v))   # [B, L, H, D] for FA
    try:
        if not want("fa4"):
            raise ImportError("skipped (ONLY)")
        from vllm.vllm_flash_attn.cute.interface import flash_attn_func
        out = flash_attn_func(qb, kb, vb)
        out = out[0] if isinstance(out, tuple) else out
        err = (out.transpose(1, 2)[0].float() - ref).abs().max().item()
        res[f"FA4 cute (vllm), bf16 O  [max|diff| vs ours {err:.2e}]"] = timeit(lambda: flash_attn_func(qb, kb, vb))
    except Exception as e:  # noqa: BLE001
        print("FA4 cute unavailable:", type(e).__name__, str(e)[:300])
    try:
        if not want("cudnn"):
            raise ImportError("skipped (ONLY)")
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            out = torch.nn.functional.scaled_dot_product_attention(q, k, v)
            err = (out[0].float() - ref).abs().max().item()
            res[f"cuDNN SDPA, bf16 O  [max|diff| vs ours {err:.2e}]"] = timeit(
                lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
    except Exception as e:  # noqa: BLE001
        print("cuDNN SDPA unavailable:", type(e).__name__, str(e)[:300])
    try:
        if not want("fa2"):
            raise ImportError("skipped (ONLY)")
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel([SDPBackend.FLASH_ATTENTION]):
            res["torch flash (FA2, mma.sync)"] = timeit(
                lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))
    except Exception as e:  # noqa: BLE001
        print("torch flash unavailable:", type(e).__name__, str(e)[:300])
    print(f"Lq {Lq} Lk {Lk} H {H} d {D}: {flops / 1e9:.1f} GFLOP per call")
    for name, (med, mn) in res.items():
        print(f"  {name:60s} median {med * 1e3:7.1f} us ({flops / med / 1e9:6.1f} TFLOP/s)  "
              f"min {mn * 1e3:7.1f} us ({flops / mn / 1e9:6.1f})")


if __name__ == "__main__":
    main()
