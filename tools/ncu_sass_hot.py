"""Per-opcode executed-instruction and stall-sample totals of an ncu report's SASS source page, plus
the hottest lines: python tools/ncu_sass_hot.py <report.ncu-rep> [top]"""
import collections
import csv
import re
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head = rows[1]
    ia, ie, iss = head.index("Source"), head.index("Instructions Executed"), head.index("Warp Stall Sampling (All Samples)")
    by_op, lines = collections.Counter(), []
    samp = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ia])
        n, s = int(r[ie] or 0), int(r[iss] or 0)
        op = m.group(2) if m else "?"
        by_op[op] += n
        samp[op] += s
        lines.append((s, n, r[0], r[ia].strip()))
    tot = sum(by_op.values())
    print(f"total warp instructions {tot}, stall samples {sum(samp.values())}")
    for op, n in by_op.most_common(top):
        print(f"  {op:14s} {n:10d} {n / tot:6.1%}  samples {samp[op]}")
    print("hottest lines (samples, executed):")
    for s, n, a, src in sorted(lines, reverse=True)[:top]:
        print(f"  {s:6d} {n:9d} {a[-5:]} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
