"""NVLink bytes per decode step of the LL exchange (run under torchrun, N >= 2). ncu cannot replay
a kernel that spins on a peer's writes (the peer does not replay with it), so the traffic is read
from the NVLink throughput counters instead (NVML field values NVLINK_THROUGHPUT_DATA_TX / RX,
KiB, summed over links; nvidia-smi nvlink -gt d as a fallback), before and after a few thousand
steps of the default bench step (C2 shape per GPU), and compared with the algorithmic bytes:
Q' sent to each peer (4 B per bf16 element in LL form: the value pair + the epoch) and every
split's (O', stats) record returned (8 B per float).
  python -m torch.distributed.run --nproc-per-node 2 tools/nvlink_bytes.py"""
import json
import os
import subprocess
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25716_b200 import capi, protocol  # noqa: E402
from paper_2605_25716_b200 import distributed as sdist  # noqa: E402


def counters(index):
    """(tx, rx) data bytes over all NVLinks of GPU `index`."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(index)
        vals = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                               nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError(f"nvml field {v.fieldId}: {v.nvmlReturn}")
            out.append(int(v.value.ullVal) * 1024)
        return tuple(out), "NVML NVLINK_THROUGHPUT_DATA_TX/RX"
    except Exception as e:  # noqa: BLE001
        txt = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True,
                             text=True).stdout
        tx = rx = 0
        for line in txt.splitlines():
            if "Tx" in line and "KiB" in line:
                tx += int(line.split(":")[-1].split()[0]) * 1024
            if "Rx" in line and "KiB" in line:
                rx += int(line.split(":")[-1].split()[0]) * 1024
        return (tx, rx), f"nvidia-smi nvlink -gt d (NVML: {e})"


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    H, D, BP = 32, 128, 16
    L = 8192 // world
    B = BP * world
    shard = protocol.KVShard(B, H, L, D, dev)
    own = protocol.DomainKeys(list(range(1, B + 1)), 0, rank + 1, H, D, dev)
    g = torch.Generator(device=dev).manual_seed(rank)
    shard.ship_segment(torch.randn((B, H, L, D), generator=g, device=dev).to(torch.bfloat16),
                       torch.randn((B, H, L, D), generator=g, device=dev).to(torch.bfloat16), own, rank * L)
    inq = [protocol.DomainKeys(list(range(rank * BP + 1, rank * BP + BP + 1)), 0, dom + 1, H, D, dev)
           for dom in range(world)]
    S = capi.default_splits(B, H, 1, L, kv_heads=H, head_dim=D)
    lld = sdist.LLDecode(BP, H, D, inq, shard, n_splits=S, kv_heads=H)
    q = torch.randn((BP, H, 1, D), generator=g, device=dev).to(torch.bfloat16)
    out = torch.empty((BP, H, 1, D), device=dev)
    for _ in range(10):
        lld.step(q, out)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        lld.step(q, out)
    steps = 2000
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    (tx0, rx0), how = counters(local)
    for _ in range(steps):
        gr.replay()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    (tx1, rx1), _ = counters(local)
    lld.check()
    peers = world - 1
    q_bytes = BP * H * D * 4 * peers                  # my Q' into every peer's slot (LL: bf16 pair + epoch)
    rec_bytes = lld.S * BP * H * (D + 2) * 8 * peers  # my domain's records into every peer inquirer's slot
    res = {"rank": rank, "world": world, "steps": steps, "splits": lld.S, "counter": how,
           "tx_bytes_per_step": (tx1 - tx0) / steps, "rx_bytes_per_step": (rx1 - rx0) / steps,
           "algorithmic_tx_bytes_per_step": q_bytes + rec_bytes,
           "algorithmic": {"q_ll": q_bytes, "records_ll": rec_bytes}}
    res["tx_over_algorithmic"] = res["tx_bytes_per_step"] / res["algorithmic_tx_bytes_per_step"]
    print(json.dumps(res), flush=True)
    dist.barrier(device_ids=[local])
    os._exit(0)


if __name__ == "__main__":
    main()
