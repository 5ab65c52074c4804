"""Per-iteration timeline of one prefill K2 CTA from a trace build of the library (compile
k2_prefill_tc.cu with -DSDA_K2_TRACE, link it into a copy of the .so, point SDA_LIB_PATH at it):
softmax wait / arrive and MMA issue times per KV tile j, in ns. This is how the S -> softmax ->
PV -> S chain of each Q tile was found to set the period (K2 prefill).
  SDA_LIB_PATH=_variants/trace/libsdattn_b200.so python tools/k2_trace.py"""
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
    base = t[0][0]
    print("MMA warp, ns relative to sm0_wait(j): top, v_full ok, pv0 issue, before k_full, k_full ok, s0 issued, pv1 issue")
    for j in range(2, 10):
        b = t[0][j]
        print(j, [int(t[k][j] - b) for k in (6, 7, 4, 9, 10, 8, 5)], "sm0_arr", int(t[2][j] - b), "sm1_arr", int(t[3][j] - b))
    print("j  sm0_wait  sm0_arr  X0   sm1_wait sm1_arr  X1   pv0_iss pv1_iss  period")
    for j in range(n):
        per = t[0][j + 1] - t[0][j] if j + 1 < n else 0
        print(f"{j:2d} {t[0][j]-base:8d} {t[2][j]-base:8d} {t[2][j]-t[0][j]:5d} {t[1][j]-base:8d} {t[3][j]-base:8d} "
              f"{t[3][j]-t[1][j]:5d} {t[4][j]-base:8d} {t[5][j]-base:8d} {per:6d}")


def main_causal():
    """causal mode (the inquirer's local span, C3): CTA (0,0,0)'s per-KV-tile stamps over its two
    segments (Q-tile pairs 7 and 0) and the (start, end) of the 32 CTAs with blockIdx.y = 0."""
    Lq, H, D = 2048, 32, 128
    dev = torch.device("cuda")
    q = torch.randn((1, H, Lq, D), device=dev).to(torch.bfloat16)
    k = torch.randn((1, H, Lq, D), device=dev).to(torch.bfloat16)
    v = torch.randn((1, H, Lq, D), device=dev).to(torch.bfloat16)
    for _ in range(3):
        ops.partial_attention_causal(q, k, v, causal_offset=0, n_splits=1)
    torch.cuda.synchronize()
    buf = np.zeros((24, 64), dtype=np.uint64)
    capi.LIB.sda_debug_k2_trace.argtypes = [ct.c_void_p]
    assert capi.LIB.sda_debug_k2_trace(buf.ctypes.data) == 0
    t = buf.astype(np.int64)
    n = int((t[0] > 0).sum())
    base = t[0][0]
    print("j  sm0_wait  sm0_arr  X0   sm1_wait sm1_arr  X1   pv0_iss pv1_iss  period (ns)")
    for j in range(n):
        per = t[0][j + 1] - t[0][j] if j + 1 < n else 0
        print(f"{j:2d} {t[0][j]-base:8d} {t[2][j]-base:8d} {t[2][j]-t[0][j]:5d} {t[1][j]-base:8d} {t[3][j]-base:8d} "
              f"{t[3][j]-t[1][j]:5d} {t[4][j]-base:8d} {t[5][j]-base:8d} {per:6d}")
    print("epilogue stamps (kind 12, per segment):", [int(t[12][i] - base) for i in range(4) if t[12][i]])
    cta = np.zeros((1024, 2), dtype=np.uint64)
    capi.LIB.sda_debug_k2_cta.argtypes = [ct.c_void_p]
    assert capi.LIB.sda_debug_k2_cta(cta.ctypes.data) == 0
    c = cta.astype(np.int64)
    n = int((c[:, 0] > 0).sum())
    c = c[:n]
    t0 = c[:, 0].min()
    print(f"{n} CTAs (y = 0): start spread {(c[:, 0].max() - t0) / 1e3:.2f} us; durations (us): "
          + " ".join(f"{(e - s) / 1e3:.1f}" for s, e in c[:8]) + f"; end max {(c[:, 1].max() - t0) / 1e3:.1f}")


def main_sk():
    """stream-K mode (one split): CTA 0's segments -- start, tile loop done, O read, ticket, end (us)."""
    Lq, Lk, H, D = 2048, 16384, int(os.environ.get("H", "32")), 128
    dev = torch.device("cuda")
    q = torch.randn((1, H, Lq, D), device=dev).to(torch.bfloat16)
    k = torch.randn((1, H, Lk, D), device=dev).to(torch.bfloat16)
    v = torch.randn((1, H, Lk, D), device=dev).to(torch.bfloat16)
    for _ in range(3):
        ops.partial_attention(q, k, v, n_splits=1)
    torch.cuda.synchronize()
    buf = np.zeros((24, 64), dtype=np.uint64)
    capi.LIB.sda_debug_k2_trace.argtypes = [ct.c_void_p]
    assert capi.LIB.sda_debug_k2_trace(buf.ctypes.data) == 0
    t = buf.astype(np.int64)
    base = t[11][0]
    print("seg  start  loop_done  O_read  ticket  end   (us from segment 0 start)")
    for si in range(8):
        if t[11][si] == 0:
            break
        print(si, [round((t[kk][si] - base) / 1e3, 2) if t[kk][si] else None for kk in (11, 12, 13, 14, 15)])
    cta = np.zeros((1024, 2), dtype=np.uint64)
    capi.LIB.sda_debug_k2_cta.argtypes = [ct.c_void_p]
    assert capi.LIB.sda_debug_k2_cta(cta.ctypes.data) == 0
    c = cta.astype(np.int64)
    n = int((c[:, 0] > 0).sum())
    c = c[:n]
    t0 = c[:, 0].min()
    end = (c[:, 1] - t0) / 1e3
    print(f"{n} CTAs: start spread {(c[:, 0].max() - t0) / 1e3:.2f} us; end min {end.min():.1f} median "
          f"{np.median(end):.1f} max {end.max():.1f} us")
    nq = 8
    for g in range(n // nq):
        e = end[g * nq:(g + 1) * nq]
        print(f"group {g:2d}: end {e.min():6.1f} .. {e.max():6.1f}  per pair: " + " ".join(f"{x:5.0f}" for x in e))
    if os.environ.get("SMID"):
        pass


if __name__ == "__main__" and not os.environ.get("PAIR"):
    main_causal() if os.environ.get("CAUSAL") else (main_sk() if os.environ.get("SK") else main())


def main_pair():
    """CTA-pair form (split grid, CTAs 0/1 = one cluster): per tile j of Q tile 0 -- the leader's
    softmax wait for PV(j-1) before its P store (16/17), the rank-1 softmax's P arrive (21) and
    its relay forwarding it (20), the MMA warp's wait for the pair's P (18 -> 19); ns from sm0_wait(j)."""
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
    print(" j  sm0_wait  pe_wait  pe_done  sm0_arr(r0)  sm0_arr(r1)  relay(r1)  mma_wait_p  mma_got_p  next sm0_wait")
    for j in range(2, 30):
        b = t[0][j]
        f = lambda k, jj=j: int(t[k][jj] - b) if t[k][jj] else -1  # noqa: E731
        print(f"{j:2d} {b - t[0][0]:9d} {f(16):8d} {f(17):8d} {f(2):11d} {f(21):11d} {f(20):10d} {f(18):11d} {f(19):10d} {int(t[0][j + 1] - b):10d}")


if __name__ == "__main__" and os.environ.get("PAIR"):
    main_pair()
