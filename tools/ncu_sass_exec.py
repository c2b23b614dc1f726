"""Executed SASS instruction mix of one kernel from an ncu source-page CSV (--page source --csv,
SASS view, optionally gzipped): warp instructions executed per opcode, and stall samples.
Usage: python tools/ncu_sass_exec.py SRC.csv[.gz] [top]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
text = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
rows = list(csv.reader(text.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex, st = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    op = r[1].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    ex[o] += int(r[ie] or 0)
    st[o] += int(r[ss] or 0)
tot, tst = sum(ex.values()), sum(st.values())
print(f"total warp instructions {tot:.4g}, stall samples {tst}")
for o, v in ex.most_common(top):
    print(f"{o:10s} {v:12d} {100.0 * v / tot:5.1f}%   stall {100.0 * st[o] / max(tst, 1):5.1f}%")
