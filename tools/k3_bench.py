"""Micro-benchmark of K3 (LSE merge + inverse permutation + unscramble), CUDA-event timed per
launch with the L2 flushed before each one (a 256 MB read: clean lines, so no write-back lands
inside the timed launch), and with the inputs L2-resident (as in a step, where K3 reads the
partials K2 has just written), for the prefill merges (C3: 1 request
x 32 heads x 2048 rows, 1 or 4 splits; C5's prefill chunk: 64 heads, 2 splits, 2 requests) and
the decode merges (16 requests x 32 heads x 1 row), per kernel form:
  tc        k3_tc_kernel (SDA_K3_TC=1; tcgen05 GEMM against the +-1 sign matrix; one key group of
            <= 2 splits + <= 1 plaintext source, q_rows >= 128; the default for >= 3 sources)
  rows      k3_rows_kernel (SDA_K3_NO_TC=1; q_rows >= 64: tables staged per CTA, scheduled gathers)
  preload   k3_merge_small_kernel (SDA_K3_NO_ROWS=1)
  pipelined k3_merge_kernel (SDA_K3_PIPELINED=1)
  python tools/k3_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops, protocol  # noqa: E402

MODES = {"default": {}, "tc": {"SDA_K3_TC": "1"}, "rows": {"SDA_K3_NO_TC": "1", "SDA_K3_ROWS": "1"}, "preload": {"SDA_K3_NO_TC": "1", "SDA_K3_NO_ROWS": "1"},
         "pipelined": {"SDA_K3_NO_TC": "1", "SDA_K3_PIPELINED": "1", "SDA_K3_NO_ROWS": "1"}}
ENVS = ("SDA_K3_TC", "SDA_K3_NO_TC", "SDA_K3_ROWS", "SDA_K3_NO_ROWS", "SDA_K3_PIPELINED")


def run(B, H, Lq, S, D=128, reps=20, out_dtype=torch.bfloat16, plain=0, kv_heads=None, identity=False):
    dev = torch.device("cuda")
    HKV = kv_heads or H
    keys = protocol.DomainKeys(list(range(1, B + 1)), 0, 1, HKV, D, dev)
    o = torch.randn((S, B, H, Lq, D), device=dev)
    st = torch.stack([torch.randn((S, B, H, Lq), device=dev), torch.rand((S, B, H, Lq), device=dev) + 0.5], -1)
    pinv = None
    if Lq > 1:
        pinv = torch.stack([torch.arange(Lq, device=dev) if identity else torch.randperm(Lq, device=dev)
                            for _ in range(B)]).to(torch.int32).contiguous()
    srcs = ops.sources_from_splits(o, st, keys.dev, pinv)
    if plain:   # the inquirer's own span (plaintext, natural row order), as bench.py's C3 / C5 steps
        lo = torch.randn((plain, B, H, Lq, D), device=dev)
        ls = torch.stack([torch.randn((plain, B, H, Lq), device=dev), torch.rand((plain, B, H, Lq), device=dev) + 0.5], -1)
        srcs = srcs + ops.sources_from_splits(lo, ls)
    out = torch.empty((B, H, Lq, D), device=dev, dtype=out_dtype)
    flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    res = {}
    for mode, env in MODES.items():
        for k in ENVS:
            os.environ.pop(k, None)
        os.environ.update(env)
        for _ in range(3):
            ops.unscramble_merge(srcs, out=out, key_heads=HKV)
        ref = out.clone()
        g = torch.cuda.CUDAGraph()   # one K3 launch, replayed: no host time inside the events
        with torch.cuda.graph(g):
            ops.unscramble_merge(srcs, out=out, key_heads=HKV)
        med = []
        for cold in (True, False):
            ts = []
            for _ in range(reps):
                if cold:
                    flush.sum()
                else:
                    g.replay()   # the inputs are in L2 from the previous launch
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            med.append(ts[len(ts) // 2])
        res[mode] = (med, ref)
    for k in ENVS:
        os.environ.pop(k, None)
    nbytes = (S + plain) * B * H * Lq * (D + 2) * 4 + B * H * Lq * D * out.element_size() + (B * Lq * 4 if Lq > 1 else 0)
    base = res["preload"][1].float()
    worst = max(float((r.float() - base).abs().max() / base.abs().max()) for _, r in res.values())
    print(f"B={B} H={H}/{HKV} Lq={Lq} S={S}+{plain} out {str(out_dtype)[6:]} ({nbytes / 1e6:.1f} MB): " +
          ", ".join(f"{m} {t[0]:.1f} us cold ({nbytes / t[0] / 1e3:.0f} GB/s) / {t[1]:.1f} us L2-warm"
                    for m, (t, _) in res.items()) +
          f"; max rel diff between forms {worst:.1e}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "perm":   # random vs identity p_q^-1 (the gather's cost)
        for ident in (False, True):
            print("identity p_q^-1" if ident else "random p_q^-1")
            run(1, 32, 2048, 1, out_dtype=torch.float32, identity=ident)
            run(1, 32, 2048, 1, out_dtype=torch.float32, plain=1, identity=ident)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "c3":   # the C3 single-source merge only (ncu captures)
        run(1, 32, 2048, 1, reps=3)
        sys.exit(0)
    run(1, 32, 2048, 1)
    run(1, 32, 2048, 1, out_dtype=torch.float32)                        # VERDICT r1 C3 target shape (<= 13 us)
    run(1, 32, 2048, 4)
    run(2, 64, 2048, 2)
    run(1, 32, 2048, 1, out_dtype=torch.float32, plain=1)               # bench.py C3 step's merge
    run(1, 64, 2048, 2, out_dtype=torch.float32, plain=1, kv_heads=8)   # bench.py C5 prefill chunk's merge
    run(1, 32, 2048, 1, D=64)
    run(16, 32, 1, 13)
    run(16, 32, 1, 4)
