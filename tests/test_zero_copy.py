"""Zero-copy host buffers at the K1 input and the K3 output: a pinned host Q read by K1 and a
pinned host O written by K3 give exactly the bytes of the device-resident form (bench.py's
end-to-end measurement uses this); a pageable host tensor is refused before any launch."""
import pytest
import torch

from paper_2605_25716_b200 import capi, ops


def test_pageable_host_tensor_refused():
    x = torch.zeros((1, 2, 4, 64), dtype=torch.bfloat16)
    keys = torch.zeros((1, 16), dtype=torch.uint8)
    with pytest.raises(ValueError, match="pinned"):
        ops.scramble(x, keys, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=x, key_heads=2)


@pytest.mark.gpu
def test_pinned_q_and_o_match_device_form():
    from paper_2605_25716_b200 import protocol

    dev = torch.device("cuda", 0)
    B, H, d, S = 3, 4, 128, 5
    keys = protocol.DomainKeys([b + 1 for b in range(B)], 0, 1, H, d, dev).dev
    g = torch.Generator(device=dev).manual_seed(11)
    q = torch.randn((B, H, 1, d), generator=g, device=dev).to(torch.bfloat16)
    qs_dev = ops.scramble(q, keys, capi.PHI_FORWARD, capi.KEYS_KQ, None, key_heads=H)
    qs_zc = torch.empty_like(qs_dev)
    ops.scramble(q.cpu().pin_memory(), keys, capi.PHI_FORWARD, capi.KEYS_KQ, None, out=qs_zc, key_heads=H)
    torch.cuda.synchronize()
    assert torch.equal(qs_dev, qs_zc)

    o = torch.randn((S, B, H, 1, d), generator=g, device=dev)
    st = torch.stack([torch.randn((S, B, H, 1), generator=g, device=dev),
                      torch.rand((S, B, H, 1), generator=g, device=dev) + 0.5], -1)
    srcs = ops.sources_from_splits(o, st.contiguous(), keys, None)
    out_dev = ops.unscramble_merge(srcs, key_heads=H)
    out_zc = torch.empty((B, H, 1, d), dtype=torch.float32).pin_memory()
    ops.unscramble_merge(srcs, out=out_zc, key_heads=H)
    torch.cuda.synchronize()
    assert torch.equal(out_dev.cpu(), out_zc)
