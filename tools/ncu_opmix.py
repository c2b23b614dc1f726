"""Dynamic SASS opcode mix (warp-level instructions executed) of one kernel in an ncu report.

Usage:  python tools/ncu_opmix.py REPORT.ncu-rep KERNEL_REGEX
"""
import csv
import re
import subprocess
import sys
from collections import Counter


def main():
    rep, regex = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    si, ie = h.index("Source"), h.index("Instructions Executed")
    ss = h.index("Warp Stall Sampling (All Samples)")
    ops, stall = Counter(), Counter()
    for r in rows[2:]:
        if len(r) != len(h) or not r[ie].isdigit():
            continue
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si])
        if not m:
            continue
        ops[m.group(1)] += int(r[ie])
        stall[m.group(1)] += int(r[ss]) if r[ss].isdigit() else 0
    tot, stot = sum(ops.values()) or 1, sum(stall.values()) or 1
    print(f"{rows[0][1][:90]}\n{tot} warp instructions executed")
    for k, v in ops.most_common(28):
        print(f"  {k:10s} {v / tot * 100:5.1f}%  stall-samples {stall[k] / stot * 100:5.1f}%")


if __name__ == "__main__":
    main()
