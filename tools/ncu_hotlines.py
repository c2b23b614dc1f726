"""Stall samples and shared-memory excess wavefronts per CUDA source line of one kernel in an
ncu report (--import-source capture): python tools/ncu_hotlines.py report.ncu-rep KERNEL_REGEX"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{sys.argv[2]}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
stall = collections.Counter()
excess = collections.Counter()
text = {}
fname = None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    key = (fname, int(r[0]))
    text[key] = r[1].strip()
    try:
        stall[key] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        excess[key] += float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0)
    except ValueError:
        pass
tot = sum(stall.values()) or 1
for key, v in stall.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 20):
    print(f"{100 * v / tot:5.1f}%  excess-wf {excess[key]:>10.0f}  {key[0]}:{key[1]:<4d} {text[key][:90]}")
