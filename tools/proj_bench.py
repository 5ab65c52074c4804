"""The scrambled QKV projection (sda_project_scramble: projection GEMM + K1 as a second GEMM in
its epilogue, one tcgen05 kernel) against the unfused form (cuBLAS x @ W^T to HBM, then K1 reading
it back), CUDA-event timed. Shapes: a 2K-token span of a Llama-7B layer (d_model 4096, 32 heads x
d128) -- the C3 span's Q, and its K / V when shipped -- and a batch of decode rows.
  python tools/proj_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, ops, protocol  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(B, rows, dm=4096, H=32, d=128):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    x = (torch.randn((B, rows, dm), generator=g, device=dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn((H * d, dm), generator=g, device=dev) / dm ** 0.5).to(torch.bfloat16)
    keys = protocol.DomainKeys(list(range(1, B + 1)), 0, 1, H, d, dev)
    perm, _ = keys.span_perms(1, 0, rows)
    out = torch.empty((B, H, rows, d), dtype=torch.bfloat16, device=dev)
    y = torch.empty((B, rows, H * d), dtype=torch.bfloat16, device=dev)
    out2 = torch.empty_like(out)

    def fused():
        ops.project_scrambled(x, w, keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ, perm, out=out)

    def unfused():   # cuBLAS projection to HBM, then K1 (row gather + scramble) reading it back
        torch.matmul(x, w.t(), out=y)
        ops.scramble(y.view(B, rows, H, d).transpose(1, 2).contiguous(), keys.dev, capi.PHI_FORWARD, capi.KEYS_KQ,
                     perm, out=out2)

    tf = timeit(fused)
    tu = timeit(unfused)
    fused()
    unfused()
    torch.cuda.synchronize()
    diff = ((out.float() - out2.float()).abs().max() / out2.float().abs().max()).item()
    flops = 2.0 * B * rows * dm * H * d
    print(f"B={B} rows={rows} d_model={dm} {H}x{d}: fused {tf * 1e3:.1f} us ({flops / tf / 1e9:.0f} TFLOP/s of "
          f"projection), cuBLAS + K1 {tu * 1e3:.1f} us ({flops / tu / 1e9:.0f}); max rel diff {diff:.1e}")


if __name__ == "__main__":
    run(1, 2048)
    run(4, 2048)
    run(16, 128)
