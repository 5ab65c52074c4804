"""Timeline of the tensor-core K1 (k1_tc_kernel) on the C3 step's batch (the span's K and V into the
cache + its Q, one launch) from the debug stamps (SDA_K1TC_TRACE=1): per CTA, clock64 at start,
first B built, and per tile: loader issues the gather (ld), the MMA warp sees the stage full (full),
MMAs issued (mma), epilogue sees the accumulator (acc), store issued (st). Thousands of SM cycles.
  python tools/k1_trace.py [n_ctas_to_print]"""
import ctypes as ct
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SDA_K1TC_TRACE"] = "1"
from paper_2605_25716_b200 import capi, ops, protocol  # noqa: E402


def main(show=3, H=32, D=128, LQ=2048, LK=16384):
    dev = torch.device("cuda")
    keys = protocol.DomainKeys([1], 0, 1, H, D, dev)
    shard = protocol.KVShard(1, H, LK + LQ, D, dev, torch.bfloat16)
    g = torch.Generator(device=dev).manual_seed(7)
    q, kn, vn = (torch.randn((1, H, LQ, D), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    pq, _ = keys.span_perms(0, LK, LQ)
    pkv, _ = keys.span_perms(1, LK, LQ)
    qs = torch.empty_like(q)
    jobs = [ops.scramble_job(kn, keys.dev, capi.PHI_INV_T, capi.KEYS_KQ, pkv, out=shard.k, out_row_offset=LK, key_heads=H),
            ops.scramble_job(vn, keys.dev, capi.PHI_FORWARD, capi.KEYS_V, pkv, out=shard.v, out_row_offset=LK, key_heads=H),
            ops.scramble_job(q, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, pq, out=qs, key_heads=H)]
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(3):
        ops.scramble_batch(jobs, D)
    flush.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.scramble_batch(jobs, D)
    e1.record()
    torch.cuda.synchronize()
    print(f"K1 batch (3 jobs, L2 flushed): {e0.elapsed_time(e1) * 1e3:.1f} us")
    n = 148
    buf = (ct.c_ulonglong * (64 * n))()
    assert capi.LIB.sda_debug_k1tc_trace(buf, n) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 64).astype(np.int64)
    names = ["start", "B"] + [f"{w}{i}" for i in range(10) for w in ("ld", "full", "mma", "acc", "st")]
    for c in range(min(show, n)):
        row = t[c]
        base = row[0]
        items = sorted(((names[i], (row[i] - base) / 1000.0) for i in range(min(64, len(names)))
                        if row[i] >= base and row[i] != 0), key=lambda x: x[1])
        print(f"CTA {c}: " + "  ".join(f"{k}={v:.1f}" for k, v in items))
    ends = [max(r[r > 0]) - r[0] for r in t if r[0] > 0]
    print(f"CTA span (kcycles): median {np.median(ends) / 1000:.1f}, max {max(ends) / 1000:.1f}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
