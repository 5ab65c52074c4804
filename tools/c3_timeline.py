"""Kernel timeline of bench.py's C3 prefill step (its run_prefill sub-measurement) from the CUDA
profiler (torch.profiler / CUPTI: device start / end of every kernel, overlaps included): per
kernel name the launches, mean duration and share, and the idle gaps between kernels.
  python tools/c3_timeline.py"""
import collections
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(bench.ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    bench.run_prefill(dev, 3, 3, peaks)   # warm
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = bench.run_prefill(dev, 5, 3, peaks)
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.name and
           "Memcpy" not in e.name and "Memset" not in e.name]
    evs.sort(key=lambda e: e.time_range.start)
    by = collections.defaultdict(list)
    for e in evs:
        by[e.name[:90]].append(e.time_range.elapsed_us())
    total = sum(sum(v) for v in by.values())
    print(f"step {res['ms_per_step'] * 1e3:.1f} us ({res['value']:.0f} TFLOP/s)")
    for name, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {len(v):4d} x {sum(v) / len(v):8.1f} us  {sum(v) / total:6.1%}  {name}")
    gaps = [evs[i + 1].time_range.start - evs[i].time_range.end for i in range(len(evs) - 1)]
    big = sorted(g for g in gaps if g > 1)
    print(f"gaps > 1 us between consecutive kernels: {len(big)}, total {sum(big):.1f} us, largest {big[-5:]}")


if __name__ == "__main__":
    main()
