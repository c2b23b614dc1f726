"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    data.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = d["Metric Value"]
agg, tot = collections.OrderedDict(), 0.0
for (_, k), m in data.items():
    dur = float(m["gpu__time_duration.sum"].replace(",", "")) / 1e3
    tot += dur
    name = k.replace("void ", "").replace("mgb::(anonymous namespace)::", "").split("(")[0]
    a = agg.setdefault(name, [0.0, 0])
    a[0] += dur
    a[1] += 1
for n, (d, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{d:10.1f} us {c:4d}x {100 * d / tot:5.1f}%  {n}")
print(f"total {tot:.1f} us over {len(data)} launches")
