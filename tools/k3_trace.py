"""Timeline of the tensor-core K3 (k3_tc_kernel) from its debug stamps (SDA_K3TC_TRACE=1): per CTA,
clock64 at kernel start, B built, and per tile: split warp 0 before / after its A-stage wait, its
rows written, the MMAs issued; epilogue warp 0 before / after the accumulator wait, tile finished.
Printed in thousands of SM cycles from the CTA's start. Shape: C3's single-source merge (f32 out).
  python tools/k3_trace.py [n_ctas_to_print]"""
import ctypes as ct
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SDA_K3TC_TRACE"] = "1"
os.environ["SDA_K3_TC"] = "1"   # the tensor-core form for every eligible merge (the default takes it for >= 3 sources)
from paper_2605_25716_b200 import capi, ops, protocol  # noqa: E402


def main(show=4, B=1, H=32, Lq=2048, S=1, D=128, plain=0, out_dtype=torch.float32):
    dev = torch.device("cuda")
    keys = protocol.DomainKeys(list(range(1, B + 1)), 0, 1, H, D, dev)
    o = torch.randn((S, B, H, Lq, D), device=dev)
    st = torch.stack([torch.randn((S, B, H, Lq), device=dev), torch.rand((S, B, H, Lq), device=dev) + 0.5], -1)
    pinv = torch.stack([torch.randperm(Lq, device=dev) for _ in range(B)]).to(torch.int32).contiguous()
    srcs = ops.sources_from_splits(o, st, keys.dev, pinv)
    if plain:
        lo = torch.randn((plain, B, H, Lq, D), device=dev)
        ls = torch.stack([torch.randn((plain, B, H, Lq), device=dev), torch.rand((plain, B, H, Lq), device=dev) + 0.5], -1)
        srcs = srcs + ops.sources_from_splits(lo, ls)
    out = torch.empty((B, H, Lq, D), device=dev, dtype=out_dtype)
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(3):
        ops.unscramble_merge(srcs, out=out, key_heads=H)
    flush.sum()
    torch.cuda.synchronize()
    ops.unscramble_merge(srcs, out=out, key_heads=H)
    torch.cuda.synchronize()
    n = 148
    buf = (ct.c_ulonglong * (64 * n))()
    assert capi.LIB.sda_debug_k3tc_trace(buf, n) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(n, 64).astype(np.int64)
    names = ["start", "B"] + [f"{w}{i}" for i in range(7) for w in ("s_wait", "s_go", "s_done", "mma", "e_wait", "e_go", "e_done", "e_ph1")]
    for c in range(min(show, n)):
        row = t[c]
        base = row[0]
        if base == 0:
            continue
        items = [(names[i], (row[i] - base) / 1000.0) for i in range(64) if row[i] >= base and row[i] != 0]
        items.sort(key=lambda x: x[1])
        print(f"CTA {c}: " + "  ".join(f"{k}={v:.1f}" for k, v in items))
    ends = [max(r[r > 0]) - r[0] for r in t if r[0] > 0]
    if not ends:
        print("no trace (the merge did not run on the tensor-core form)")
        return
    print(f"CTA span (kcycles): median {np.median(ends) / 1000:.1f}, max {max(ends) / 1000:.1f}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
    print("-- with a plaintext source (bench.py C3 merge)")
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4, plain=1)
