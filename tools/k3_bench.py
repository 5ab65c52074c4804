"""Micro-benchmark of K3 (LSE merge + inverse permutation + unscramble), CUDA-event timed:
the prefill merge (1 request x 32 heads x 2048 rows, 4 splits, p_q^-1 gather) and the decode
merge (16 requests x 32 heads x 1 row, 10 splits), for the preloading and the pipelined kernel.
  python tools/k3_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops, protocol  # noqa: E402


def run(B, H, Lq, S, D=128, reps=20):
    dev = torch.device("cuda")
    keys = protocol.DomainKeys(list(range(1, B + 1)), 0, 1, H, D, dev)
    o = torch.randn((S, B, H, Lq, D), device=dev)
    st = torch.stack([torch.randn((S, B, H, Lq), device=dev), torch.rand((S, B, H, Lq), device=dev) + 0.5], -1)
    pinv = None
    if Lq > 1:
        pinv = torch.stack([torch.randperm(Lq, device=dev) for _ in range(B)]).to(torch.int32).contiguous()
    srcs = ops.sources_from_splits(o, st, keys.dev, pinv)
    out = torch.empty((B, H, Lq, D), device=dev)
    res = {}
    for mode in ("preload", "pipelined"):
        if mode == "pipelined":
            os.environ["SDA_K3_PIPELINED"] = "1"
        else:
            os.environ.pop("SDA_K3_PIPELINED", None)
        for _ in range(3):
            ops.unscramble_merge(srcs, out=out, key_heads=H)
        ref = out.clone()
        g = torch.cuda.CUDAGraph()   # replayed: no host launch overhead in the small cases
        with torch.cuda.graph(g):
            for _ in range(reps):
                ops.unscramble_merge(srcs, out=out, key_heads=H)
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[mode] = (e0.elapsed_time(e1) / reps * 1e3, ref)
    nbytes = S * B * H * Lq * (D + 2) * 4 + B * H * Lq * D * 4
    same = torch.equal(res["preload"][1], res["pipelined"][1])
    print(f"B={B} H={H} Lq={Lq} S={S}: " + ", ".join(f"{m} {t:.1f} us ({nbytes / t / 1e3:.0f} GB/s)"
                                                     for m, (t, _) in res.items()) + f", identical: {same}")


if __name__ == "__main__":
    run(1, 32, 2048, 4)
    run(1, 32, 2048, 1)
    run(16, 32, 1, 10)
    run(16, 32, 1, 4)
    run(2, 64, 2048, 2)
