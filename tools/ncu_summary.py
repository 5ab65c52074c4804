"""Summarise ncu output into profiles/: a launch list CSV (gpu__time_duration per launch) and/or
a --set full report (.ncu-rep). Prints markdown and writes JSON next to the target.

  python tools/ncu_summary.py launches gpurun_out/launches_r01.csv profiles/launches_r01.json
  python tools/ncu_summary.py report   gpurun_out/k2_r01.ncu-rep   profiles/k2_decode_r01.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu.sum",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard", "lts__t_bytes.sum",
           "sm__memory_throughput.avg.pct_of_peak_sustained_elapsed"]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", "nsecond"), 1e-9)
            agg.setdefault(name, []).append(v)
    total = sum(sum(v) for v in agg.values())
    out = []
    for k, v in agg.items():
        out.append({"kernel": k, "launches": len(v), "mean_us": 1e6 * sum(v) / len(v), "share": sum(v) / total})
    return out


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                val = r[i].replace(",", "")
                try:
                    val = float(val) * UNIT.get(units[i], 1)
                except ValueError:
                    pass
                d[m] = val
        res.append(d)
    return res


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    data = launches(src) if kind == "launches" else report(src)
    json.dump(data, open(dst, "w"), indent=1)
    for d in data:
        print(json.dumps(d))
