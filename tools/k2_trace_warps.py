"""Per-warp P hand-off times of Q tile 0 in a K2 prefill trace build (-DSDA_K2_TRACE; split grid,
CTA 0): for each key tile j, ns from softmax warp 0 getting S0(j) to each of warps 0-3 announcing
P0(j) (p_full completes with the last of them), and the period.
  SDA_LIB_PATH=_variants/trace/libsdattn_b200.so python tools/k2_trace_warps.py"""
import ctypes as ct
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops  # noqa: E402


def main():
    Lq, Lk, H, S, D = 2048, 16384, 32, 4, 128
    dev = torch.device("cuda")
    q = torch.randn((1, H, Lq, D), device=dev).to(torch.bfloat16)
    k = torch.randn((1, H, Lk, D), device=dev).to(torch.bfloat16)
    v = torch.randn((1, H, Lk, D), device=dev).to(torch.bfloat16)
    for _ in range(3):
        ops.partial_attention(q, k, v, n_splits=S)
    torch.cuda.synchronize()
    buf = np.zeros((24, 64), dtype=np.uint64)
    capi.LIB.sda_debug_k2_trace.argtypes = [ct.c_void_p]
    assert capi.LIB.sda_debug_k2_trace(buf.ctypes.data) == 0
    t = buf.astype(np.int64)
    n = int((t[0] > 0).sum())
    print("j   P0 by warp0 warp1 warp2 warp3 (ns after S0(j))   last-first   period")
    lasts = []
    for j in range(n):
        b = t[0][j]
        a = [t[k][j] - b for k in (2, 18, 19, 20)]
        per = t[0][j + 1] - b if j + 1 < n else 0
        lasts.append(int(np.argmax(a)))
        print(j, " ".join(f"{int(x):6d}" for x in a), f"{int(max(a) - min(a)):6d}", f"{int(per):6d}")
    print("last warp counts:", {w: lasts.count(w) for w in range(4)})


if __name__ == "__main__":
    main()
