"""Multi-GPU exchange check (needs >= 2 visible GPUs, else skipped): tools/exchange_check.py under
torchrun -- the decode step through NCCL all-to-all, through the peer-memory push/wait kernels
(bit-identical) and through the LL-chained kernels (same math, <= 1e-5 relative), eager and from
a CUDA graph, over 30 steps."""
import os
import re
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_exchange_check_two_gpus():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tools", "exchange_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=500)
    # the two ranks print concurrently: their lines can interleave without a newline
    lines = re.findall(r"rank \d+: .*?\((?:ok|FAIL)\)", r.stdout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert len(lines) == 2 and all("True" in ln and "(ok)" in ln for ln in lines), lines
