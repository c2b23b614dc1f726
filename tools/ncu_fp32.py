"""Per-launch summary of an ncu --set full capture (raw page CSV): duration, DRAM bytes, and
EXECUTED FP32 flops from the SASS counters (fadd + fmul + 2 ffma thread instructions per
elapsed cycle x elapsed cycles), with HBM and FP32 fractions.
Usage: python tools/ncu_fp32.py RAW.csv.gz [hbm_peak_gbs] [--json out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ncu_csv import raw_rows  # noqa: E402

FP32_PEAK = 148 * 128 * 2 * 1.965e9


def val(r, k):
    v = r.get(k, "")
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rows = raw_rows(sys.argv[1])
    hbm = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 6549.1
    hdr, units, data = rows[0], rows[1], rows[2:]
    recs = [dict(zip(hdr, r)) for r in data]
    out = []
    for r in recs:
        name = r.get("Kernel Name", "")
        dur_ns = val(r, "gpu__time_duration.sum")
        unit = units[hdr.index("gpu__time_duration.sum")]
        dur_s = dur_ns * (1e-9 if unit == "ns" else 1e-6 if unit in ("us", "usecond") else 1e-3 if unit in ("ms", "msecond") else 1e-9)
        cyc = val(r, "smsp__cycles_elapsed.avg")
        nsmsp = 148 * 4
        per = lambda op: val(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
        flops = (per("fadd") + per("fmul") + 2 * per("ffma")) * cyc
        dflops = (per("dadd") + per("dmul") + 2 * per("dfma")) * cyc
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        bu = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
        rd, wr = rd * scale, wr * scale
        out.append({"kernel": name[:90], "us": dur_s * 1e6, "dram_bytes": rd + wr,
                    "hbm_frac": (rd + wr) / dur_s / (hbm * 1e9) if dur_s else 0,
                    "fp32_flops_exec": flops, "fp32_frac": flops / dur_s / FP32_PEAK if dur_s else 0,
                    "fp64_flops_exec": dflops, "regs": val(r, "launch__registers_per_thread"),
                    "occ_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                    "ipc": val(r, "sm__inst_executed.avg.per_cycle_active")})
    for o in out:
        print(f"{o['us']:9.1f} us  dram {o['dram_bytes']/1e6:9.1f} MB  hbm {o['hbm_frac']:.2f}  fp32 {o['fp32_flops_exec']/1e9:8.2f} GF "
              f"({o['fp32_frac']:.3f})  fp64 {o['fp64_flops_exec']/1e9:6.2f} GF  regs {o['regs']:.0f} occ {o['occ_pct']:.0f}% ipc {o['ipc']:.2f}  {o['kernel'][:60]}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
