"""Timeline of the split-row K2 form (SDA_K2_HELP=1) from a trace build (-DSDA_K2_TRACE): per key
tile j of CTA 0, ns relative to the primary group-0 warp getting S(j): primary max exchange done,
primary P (keys 0-63) arrive, helper got S, helper P (keys 64-127) arrive, PV0 issue; then the
same for group 1 and the period.
  SDA_LIB_PATH=_variants/help_trace/libsdattn_b200.so python tools/k2_trace_help.py"""
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
    print("j   xch0 parr0 hwait0 harr0 pv0 | s1wait parr1 hwait1 harr1 pv1 | period")
    for j in range(n):
        b = t[0][j]
        per = t[0][j + 1] - b if j + 1 < n else 0
        r = [t[k][j] - b for k in (20, 2, 18, 19, 4)] + [t[k][j] - b for k in (1, 3, 22, 23, 5)]
        print(j, " ".join(f"{int(x):6d}" for x in r), f"| {int(per):6d}")


if __name__ == "__main__":
    main()
