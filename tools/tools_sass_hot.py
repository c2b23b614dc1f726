"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep, regex = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}", "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ss = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(h) and r[ss].isdigit()]
tot = sum(int(r[ss]) for r in body) or 1
print(f"total samples {tot}, instructions {len(body)}")
for r in sorted(body, key=lambda r: -int(r[ss]))[:n]:
    print(f"{int(r[ss]) / tot * 100:5.1f}%  {r[si].strip()[:90]}")
