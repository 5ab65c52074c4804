"""The reference's own provider tests (test_model.cpp:90-129) through the reference-side
adapter gpu_scrambled_attn (integration/), and the causal plaintext shard of the C ABI."""
import os
import subprocess

import numpy as np
import pytest
import torch

from oracle import C
from paper_2605_25716_b200 import ops
from tests.gpu_helpers import dev, gauss, max_abs_rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_model_gpu")


@pytest.mark.skipif(not os.path.exists(BIN), reason="integration binary not built (needs /root/reference)")
def test_reference_model_tests_through_adapter():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("offset", [0, 3, -2])
def test_causal_plaintext_shard(offset):
    """AttentionMask::causal(offset) (attention.hpp:25-27): key j visible to row i iff j <= i + offset."""
    lq, lk, d = 7, 10, 64
    q, k, v = gauss(61, (1, 2, lq, d)), gauss(62, (1, 2, lk, d)), gauss(63, (1, 2, lk, d))
    o, st = ops.partial_attention_causal(dev(q, torch.float32), dev(k, torch.float32), dev(v, torch.float32), offset)
    o, st = o.double().cpu().numpy()[0], st.double().cpu().numpy()[0]
    for h in range(2):
        ro, rm, rs = C.shard_attention(q[0, h], k[0, h], v[0, h], offset)
        live = rs > 0
        assert np.array_equal(st[0, h, :, 1] > 0, live)       # fully masked rows: exp_sum = 0
        assert max_abs_rel(o[0, h][live], ro[live]) < 1e-4
        assert np.allclose(st[0, h, live, 0], rm[live], atol=1e-5)
