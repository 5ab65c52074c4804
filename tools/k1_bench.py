"""Micro-benchmark of K1 (scramble + permute into the cache): tcgen05 vs SIMT, random vs
identity token permutation. CUDA-event timed, L2 flushed between launches by a 256 MB read
(clean lines: a write flush would leave dirty lines whose write-back lands in the timed launch).
  python tools/k1_bench.py [B H rows d]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops  # noqa: E402


def main():
    B, H, L, D = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (16, 32, 8192, 128)))
    dev = torch.device("cuda")
    kh = [capi.negotiate_keyset(capi.shared_seed(1, b + 1), b + 1, 0, 1, H, D) for b in range(B)]
    kd = ops.upload_keys([k.pack() for k in kh], dev)
    x = torch.randn((B, H, L, D), device=dev).to(torch.bfloat16)
    out = torch.empty_like(x)
    perm_rand = ops.upload_perms([k.span_perm(1, 0, L) for k in kh], dev)
    perm_id = ops.upload_perms([np.arange(L, dtype=np.uint32)] * B, dev)
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    nbytes = 2 * x.numel() * 2
    for impl in ("tc", "simt"):
        if impl == "simt":
            os.environ["SDA_K1_SIMT"] = "1"
        else:
            os.environ.pop("SDA_K1_SIMT", None)
        for name, perm in (("random", perm_rand), ("identity", perm_id), ("none", None)):
            ts = []
            for i in range(8):
                flush.sum()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ops.scramble(x, kd, capi.PHI_INV_T, capi.KEYS_KQ, perm, out=out, key_heads=H)
                e1.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            t = float(np.median(ts))
            print(f"K1 {impl:4s} perm={name:8s} B{B} H{H} L{L} d{D}: {t * 1e3:8.1f} us  {nbytes / t / 1e6:7.1f} GB/s")


if __name__ == "__main__":
    main()
