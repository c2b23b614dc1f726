"""Serialized per-kernel-family cost of one bench step from an ncu launch list
(--metrics gpu__time_duration.sum): python tools/ncu_breakdown.py launches.csv [launches_per_step]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
data = rows[h + 1:]
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
KEYS = ("rows_conv_fk", "rows_conv_pair", "rows_conv", "rows_spec", "cols_fwd<9, 2", "cols_fwd<9, 0",
        "cols_fwd<9, 1", "cols_inv", "eq_conv", "dyn_scan<0", "dyn_scan<1", "pointwise", "reverb_ir",
        "eq_response_basis", "eq_mag_tiles", "delay_taps", "eq_design", "eq_response", "eq_mags", "param_gather")
ALIAS = {"cols_fwd<9, 2": "cols_fwd<delay taps>", "cols_fwd<9, 0": "cols_fwd<kernel>",
         "cols_fwd<9, 1": "cols_fwd<signal>", "dyn_scan<0": "dyn_scan<compressor>", "dyn_scan<1": "dyn_scan<gate>"}


def fam(name):
    for k in KEYS:
        if k in name:
            return ALIAS.get(k, k)
    return name[:40]


t, c = collections.Counter(), collections.Counter()
for r in data[-n:]:
    v = float(r[vi].replace(",", ""))
    f = fam(r[ki])
    t[f] += v
    c[f] += 1
tot = sum(t.values())
for f, v in t.most_common():
    print(f"{f:24s} {v / 1e6:8.2f} ms {c[f]:5d} launches {100 * v / tot:5.1f}%")
print(f"total {tot / 1e6:.2f} ms serialized over {sum(c.values())} launches")
