"""profiles/r02s_traffic.json from ncu --set full captures of a config-5 union (raw page CSVs):
per kernel family (bench.kernel_family), DRAM bytes (read + write) per launch averaged over the
captured launches, and their count. bench.py reports the dominant family's figure as
roofline.traffic. Usage: python tools/traffic_json.py OUT.json RAW.csv.gz [RAW2.csv.gz ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from _ncu_csv import raw_rows  # noqa: E402
from bench import kernel_family  # noqa: E402

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
fam = {}
for path in sys.argv[2:]:
    rows = raw_rows(path)
    hdr, units = rows[0], rows[1]
    ki, rd, wr, du = (hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                              "gpu__time_duration.sum"))
    for r in rows[2:]:
        f = kernel_family(r[ki])
        f = "pointwise" if f.startswith("pointwise") else f
        b = float(r[rd].replace(",", "")) * SCALE.get(units[rd], 1) + float(r[wr].replace(",", "")) * SCALE.get(units[wr], 1)
        d = fam.setdefault(f, {"dram_bytes": 0.0, "launches": 0, "us": 0.0})
        d["dram_bytes"] += b
        d["launches"] += 1
        d["us"] += float(r[du].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(units[du], 1.0)
out = {k: {"dram_bytes_per_launch": v["dram_bytes"] / v["launches"], "launches_captured": v["launches"],
           "us_per_launch_ncu": v["us"] / v["launches"]} for k, v in fam.items()}
out["_source"] = ("ncu --set full --clock-control none, one config-5 union render (tools/c5_one_union.py), "
                  "cold serialized launches: " + ", ".join(os.path.basename(p) for p in sys.argv[2:]))
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
