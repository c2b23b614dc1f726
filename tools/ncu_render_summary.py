"""Summarise an ncu --set full capture of one render into profiles/.

Usage:  python tools/ncu_render_summary.py gpurun_out/prof_render.ncu-rep profiles/r01
Writes <prefix>_ncu_kernels.csv (one row per launch) and <prefix>_ncu_summary.md, and
updates profiles/traffic.json: DRAM bytes (read + write) per render step type, summed over
the step's kernels of the FIRST render in the capture (cold L2: upper bound on traffic).
"""
import csv
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _ncu_csv import raw_rows  # noqa: E402

KEYS = {
    "dur_us": "gpu__time_duration.sum",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "fp32_inst": "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
}

# kernel-name fragment -> step type (the step whose work the kernel does)
STEP_OF = [("eq_", "eq"), ("dyn_scan<false", "compressor"), ("dyn_scan<true", "noisegate"),
           ("reverb_ir", "reverb"), ("delay_", "delay"), ("pointwise_vec4<(mgb::PointOp)0>", "copy"),
           ("pointwise_vec4<(mgb::PointOp)1>", "gain"), ("pointwise_vec4<(mgb::PointOp)2>", "imager")]


def to_num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
    return x * scale


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    rows = raw_rows(rep)
    head, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(head)}
    recs = []
    for r in rows[2:]:
        rec = {"id": int(r[col["ID"]]), "kernel": r[col["Kernel Name"]]}
        for k, m in KEYS.items():
            if m in col:
                rec[k] = to_num(r[col[m]], units[col[m]])
        recs.append(rec)
    with open(prefix + "_ncu_kernels.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["id", "kernel"] + list(KEYS))
        w.writeheader()
        for rec in recs:
            w.writerow(rec)
    lines = ["| id | kernel | us | regs | grid | occ % | IPC | DRAM rd MB | DRAM wr MB | L2 hit % |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in recs:
        name = r["kernel"].replace("mgb::(anonymous namespace)::", "").replace("void ", "")[:48]
        lines.append(f"| {r['id']} | `{name}` | {r['dur_us']:.1f} | {r['regs']:.0f} | {r['grid']:.0f} | "
                     f"{r['occ_pct']:.0f} | {r['ipc']:.2f} | {r['dram_rd'] / 1e6:.1f} | {r['dram_wr'] / 1e6:.1f} | "
                     f"{r['l2_hit_pct']:.0f} |")
    with open(prefix + "_ncu_summary.md", "w") as f:
        f.write("# ncu --set full, one config-2 render (cold caches, serialised replays)\n\n")
        f.write("Absolute durations are replay-serialised and cold; compare shares. Source: "
                f"`{os.path.basename(rep)}` (gpurun_out/, not committed).\n\n")
        f.write("\n".join(lines) + "\n")
    # Traffic per render step type over the first render in the capture: from the first
    # render's first kernel up to the next render's. Conv kernels are attributed by
    # order: a prologue pair (cols_fwd<.., 0>, rows_spec) belongs to the reverb_ir / delay_dense
    # that precedes it; main triples (cols_fwd<.., 1>, rows_conv, cols_inv) follow the step
    # order reverb then delay (config 2's type string ...rd...).
    # the render's first kernel: the EQ magnitude tiles (basis path) or eq_conv<1> (split EQ)
    first = lambda k: "eq_mag_tiles" in k or "eq_conv<1>" in k or "eq_conv<1," in k  # noqa: E731
    start = next(i for i, r in enumerate(recs) if first(r["kernel"]))
    end = next((i for i in range(start + 1, len(recs)) if first(recs[i]["kernel"]) or "mgb::" not in recs[i]["kernel"]),
               len(recs))
    traffic, per_kernel = {}, []
    owner, main_seen = None, 0
    for r in recs[start:end]:
        k = r["kernel"]
        b = (r["dram_rd"] or 0) + (r["dram_wr"] or 0)
        if "reverb_ir" in k:
            owner = "reverb"
        if "delay_" in k:
            owner = "delay"
        if "eq_" in k:
            step = "eq"
        elif "dyn_scan<0" in k:
            step = "compressor"
        elif "dyn_scan<1" in k:
            step = "noisegate"
        elif "pointwise_vec4<0" in k or "pointwise_wide<0" in k:
            step = "mix/out"
        elif "pointwise_vec4<1" in k:
            step = "gain"
        elif "pointwise_vec4<2" in k:
            step = "imager"
        elif "pointwise_chain" in k:
            step = "imager+gain+out (fused chain)"
        elif "reverb_ir" in k or "delay_" in k or "rows_spec" in k or ", 0>(" in k:
            step = owner
        elif "cols_fwd" in k or "rows_conv" in k or "cols_inv" in k:
            step = "reverb" if main_seen < 3 else "delay"
            main_seen += 1
        else:
            continue
        traffic[step] = traffic.get(step, 0.0) + b
        per_kernel.append({"id": r["id"], "kernel": k[:80], "step": step, "dram_bytes": b, "dur_us": r["dur_us"]})
    path = os.path.join(os.path.dirname(prefix), "traffic.json")
    with open(path, "w") as f:
        json.dump({"source": os.path.basename(prefix) + "_ncu_kernels.csv",
                   "unit": "DRAM bytes (read + write) per render, cold caches (ncu replay)",
                   "by_step_type": traffic, "kernels": per_kernel}, f, indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
