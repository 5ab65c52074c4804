"""Debug aid: K2 prefill (tensor-core form) against a torch f32 reference, per output row --
prints which rows of which (request, head, split) are off. Runs a few shapes (split grid and
stream-K, one or two Q tiles per unit).
  [SDA_K2_PSMEM=0] python tools/k2_rows_check.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import ops  # noqa: E402


def ref_split(q, k, v, a, e):
    s = (q.float() @ k[a:e].float().T) / 128 ** 0.5
    return torch.softmax(s, -1) @ v[a:e].float()


def check(lq, cap, kv_len, n_splits, hq, hkv):
    B, d = len(kv_len), 128
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((B, hq, lq, d), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((B, hkv, cap, d), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((B, hkv, cap, d), generator=g, device="cuda").to(torch.bfloat16)
    o, st = ops.partial_attention(q, k, v, torch.tensor(kv_len, dtype=torch.int32, device="cuda"), n_splits=n_splits)
    torch.cuda.synchronize()
    G = hq // hkv
    bad = 0
    for b in range(B):
        ntile = -(-kv_len[b] // 128)
        tps = -(-ntile // n_splits)
        for h in range(hq):
            for s in range(n_splits):
                a, e = s * tps * 128, min(kv_len[b], (s + 1) * tps * 128)
                if a >= e:
                    continue
                r = ref_split(q[b, h], k[b, h // G], v[b, h // G], a, e)
                err = (o[s, b, h].float() - r).abs().amax(-1) / r.abs().amax()
                rows = torch.nonzero(err > 1e-2).flatten().tolist()
                if rows:
                    bad += 1
                    print(f"  b{b} h{h} s{s}: {len(rows)} bad rows, first {rows[:8]} last {rows[-4:]}, max err {err.max().item():.3f}")
    print(f"lq {lq} cap {cap} kv_len {kv_len} splits {n_splits} hq {hq} hkv {hkv}: {'OK' if not bad else f'{bad} bad (b,h,s)'}")


SHAPES = [(128, 1024, [1024], 1, 2, 2), (256, 1024, [1024], 1, 2, 2), (256, 1024, [1024], 2, 2, 2),
          (300, 1000, [1000, 517], 3, 4, 2), (300, 1000, [1000, 517], 1, 4, 2), (512, 2048, [2048], 1, 4, 4),
          # CTA-pair shapes (whole 256-row pairs, an even pair count / stream-K group)
          (512, 1024, [1024], 2, 2, 2), (1024, 4096, [4096, 3000], 1, 4, 4), (1024, 2000, [2000, 77], 3, 4, 2),
          (2048, 16384, [16384], 1, 32, 32)]

if __name__ == "__main__":
    for args in (SHAPES[int(sys.argv[1]):] if len(sys.argv) > 1 else SHAPES):
        check(*args)
