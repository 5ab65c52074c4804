"""Print the headline metrics and the non-trivial warp-stall reasons of an ncu report's kernels
(ncu -i <rep> --page raw --csv).  python tools/ncu_summary.py <report.ncu-rep>"""
import csv
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[head.index("Kernel Name")][:100])
        for n, u, v in zip(head, units, r):
            if n in KEYS:
                print(f"  {n} = {v} {u}")
        stalls = []
        for n, v in zip(head, r):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if x > 0.1:
                    stalls.append((x, n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("  stalls/issue: " + ", ".join(f"{k} {x:.2f}" for x, k in sorted(stalls, reverse=True)))


if __name__ == "__main__":
    main(sys.argv[1])
