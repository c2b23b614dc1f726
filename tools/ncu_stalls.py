"""Stall breakdown (warps stalled per issued instruction, by reason) per launch of an ncu report.

Usage:  python tools/ncu_stalls.py REPORT.ncu-rep [ID ...]
"""
import csv
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ncu_csv import raw_rows  # noqa: E402


def main():
    rep, ids = sys.argv[1], set(sys.argv[2:])
    rows = raw_rows(rep)
    h = rows[0]
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    for r in rows[2:]:
        if ids and r[h.index("ID")] not in ids:
            continue
        st = {}
        for i, n in enumerate(h):
            if n.startswith(pre) and n.endswith(suf):
                try:
                    st[n[len(pre):-len(suf)]] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        top = sorted(st.items(), key=lambda x: -x[1])[:7]
        print(r[h.index("ID")], r[h.index("Kernel Name")].replace("mgb::<unnamed>::", "")[:34], "|",
              " ".join(f"{k}={v:.2f}" for k, v in top))


if __name__ == "__main__":
    main()
