#!/usr/bin/env python
"""Benchmark: node-samples/s and graph renders/s of the batched render path (BASELINE.json).

Headline workload (the largest single-GPU BASELINE config, config 5): 512 random mixing
consoles (generate_console(K_i in [4, 32], p = 0.3), the reference's generator, bit-identical;
random_legal_params per graph), stereo 2^17 samples at 44.1 kHz, B = 1, sources from a 64-row
uniform_noise bank (input k of a union takes row k % 64). The set is sharded over the ranks by
LPT on node-sample cost (graphs are independent: no collective on the data path) and every
rank renders its shard as unions of <= 64 consoles. A step = one render of all 512 graphs
(every processor of every node, no skipped work).

  value  — device time: each union's render captured as one CUDA graph, inputs resident in
           HBM, all unions replayed back to back; CUDA events on the replay stream around each
           step, max over ranks (barrier + synchronize on both sides). The working set (the
           arenas, ~60 GB) is far larger than L2, so no flush is needed between steps.
  e2e    — the same 512 graphs through the public API with HOST buffers (BatchRenderer /
           mg_batch_submit: pinned fp32 sources per input node, original-order parameter
           tables, device reorder, render, output D2H), host<->device copies inside the timed
           region; wall clock, max over ranks. Bytes per step are counted from the copies.
  scaling — "strong": the 512 graphs are split over N ranks.

--impl reference times the reference's own CPU renderer (oracle/_ref: the unmodified reference
compiled with the FFTW-API stand-in) on the box's host cores, one process per core, each step
a bounded sample of the same 512-graph set. Secondary lines (config 2, 3, 4, config 5's
optimisation step) ride along under their own keys at N = 1.

--backend gloo runs the N > 1 path with gloo (CPU-side timing reductions) and lets ranks share
GPUs (rank r on cuda:(r mod devices)): for exercising multi-rank code on one GPU, not for
scaling numbers.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402

L = wl.L2
FS = wl.FS
METRIC = "node-samples/sec"
UNIT = "node-samples/s"
CHUNK = 64  # consoles per union (one plan, one arena, one CUDA graph)
WORKLOAD = ("config5: 512 random consoles (generate_console K in [4,32], p=0.3, fixed topology), stereo 2^17 @ "
            "44.1 kHz, B=1, LPT-sharded over ranks, unions of <= 64 consoles per rank")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    p.add_argument("--no-extras", action="store_true", help="skip the secondary config lines")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # nominal CUDA-core FP32 at the max SM clock


class ClockSampler:
    """NVML clocks and throttle reasons sampled every 2 ms while the timed region runs."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_setup():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---- the config-5 workload -----------------------------------------------------------------

def config5_shard(rank, world):
    """(graphs, my graph indices, unions of <= CHUNK of them) for this rank."""
    from paper_2408_03204_b200 import sharding
    graphs = wl.config5_graphs()
    mine = sharding.lpt_shards([sharding.graph_cost(t, L) for t, _ in graphs], world)[rank]
    return graphs, mine, [mine[i:i + CHUNK] for i in range(0, len(mine), CHUNK)]


def union_case(mg, graphs, idx):
    """Union plan of graphs[idx] with the members' own parameter tables (concat_params order)."""
    from paper_2408_03204_b200 import sharding
    members = [graphs[i] for i in idx]
    t, e = sharding.union_arrays(members)
    rd = mg.compute_render_data_arrays(t, e)
    params = wl.union_params([m[0] for m in members], [wl.config5_member_params(i, graphs[i][0]) for i in idx])
    return t, rd, params


def node_samples(t, length=L, batch=1):
    return (len(t) - int(np.sum(np.asarray(t) == 0))) * length * batch


# ---- roofline of the kernels as they run inside the render ---------------------------------

def kernel_family(name):
    if "dyn_stream" in name:  # the streaming variant of the dynamics scan
        return "dyn_scan"
    if "rows_conv_pair" in name:  # row passes of delay / reverb items sharing a signal spectrum
        return "rows_conv_fk"
    if "delay_cols" in name:  # the delay kernel's column stage as a sparse direct DFT
        return "delay_cols"
    for key in ("rows_conv_fk", "rows_conv", "rows_spec", "cols_fwd", "cols_inv", "eq_conv", "dyn_scan",
                "pointwise_wide", "pointwise_chain", "pointwise", "reverb_ir", "eq_basis_product", "eq_mag_tiles",
                "delay_taps", "eq_design", "eq_response", "eq_mags", "param_gather"):
        if key in name:
            return key
    return name.split("(")[0][-40:]


def in_render_kernel_times(replay):
    """CUPTI (torch.profiler) trace of one replay: per kernel family, total device time (us),
    launches and the wall span of the replay; kernels inside CUDA graphs are reported one by
    one with their in-render (concurrent) durations."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        replay()
        torch.cuda.synchronize()
    fam, t0, t1 = {}, None, None
    for ev in prof.events():
        if ev.device_type.name != "CUDA" or "memset" in ev.name.lower() or "memcpy" in ev.name.lower():
            continue
        d = fam.setdefault(kernel_family(ev.name), {"us": 0.0, "launches": 0})
        d["us"] += ev.time_range.end - ev.time_range.start
        d["launches"] += 1
        t0 = ev.time_range.start if t0 is None else min(t0, ev.time_range.start)
        t1 = ev.time_range.end if t1 is None else max(t1, ev.time_range.end)
    return fam, (t1 - t0) if t0 is not None else None


def family_work(mg, procs, rd, length, batch=1):
    """Algorithmic work per render of `rd` by kernel family:
    FFT families -> ("fp32", flops of the implemented transforms, 5 N log2 N per N-point
    complex transform plus 8 flops per point of every spectral product); gather / scan /
    pointwise families -> ("hbm", bytes: every gathered row read once, every stored row written
    once, 8 B per stereo sample; a scan step's fused pointwise followers are counted with the
    pointwise family).
      reverb / delay, per (slot, batch, segment) item of the N = N1 N2 segmented transform:
        cols_fwd  column halves of the signal forward (not for items reusing the previous
                  step's spectrum, rd.shared_pairs) and of the reverb kernel spectrum (per slot)
        delay_cols the delay kernel's column stage (sparse direct DFT): HBM, its 8 N B write
        rows_conv row halves of the forward and inverse + product (rows_conv_fk: + the kernel's
                  row half per item; otherwise rows_spec does it once per slot)
        cols_inv  column half of the inverse
      eq_conv: per overlap-save window a forward and an inverse 8192-point (4096 when the step
        is too small to fill the GPU) transform + product.
    Steps computed in another step's launch (rd.step_owners: fused pointwise runs, scan
    epilogues) are counted with that launch's family, followers as writes only."""
    out = {}

    def add(k, bound, v):
        b, w = out.get(k, (bound, 0.0))
        out[k] = (bound, w + v)

    nsm = 148
    owner = rd.step_owners(batch, length)
    pairs = rd.shared_pairs(procs, batch, length)
    fam_of = {mg.NodeType.COMPRESSOR: "dyn_scan", mg.NodeType.NOISEGATE: "dyn_scan"}
    for k, st in enumerate(rd.steps):
        slots = st.store_end - st.store_begin
        t = st.type
        hbm = 8.0 * length * batch * (len(st.gather) + slots)
        if owner[k] != k and rd.steps[owner[k]].type in fam_of:
            # pointwise follower computed in a scan's epilogue: it only writes its rows
            add("dyn_scan", "hbm", 8.0 * length * batch * slots)
        elif owner[k] != k:
            add("pointwise", "hbm", 8.0 * length * batch * slots)
        elif t in (mg.NodeType.REVERB, mg.NodeType.DELAY):
            taps = procs.reverb_length if t == mg.NodeType.REVERB else procs.delay_span
            g = mg.conv_geometry(length, taps)
            n, l1, l2 = 1 << g["log_n"], g["log_n1"], g["log_n2"]
            per = batch * g["nseg"]
            items = slots * per
            shared = int(pairs[k]) * per  # items reusing step k-1's signal spectra
            sparse = t == mg.NodeType.DELAY and l1 >= 8 and mg.fft_precision() == 32
            if sparse:  # delay_cols: writes the column-stage spectrum, a few terms per output
                add("delay_cols", "hbm", slots * n * 8.0)
            add("cols_fwd", "fp32", (items - shared + (0 if sparse else slots)) * 5.0 * n * l1)
            add("cols_inv", "fp32", items * 5.0 * n * l1)
            if 8.0 * slots * n > (64 << 20):  # conv_fuse: kernel rows transformed per item
                # a shared pair (this item + its partner in step k-1) runs 5 row transforms, not 6
                add("rows_conv_fk", "fp32", items * (3 * 5.0 * n * l2 + 16.0 * n) - shared * 5.0 * n * l2)
            else:
                add("rows_spec", "fp32", slots * 5.0 * n * l2)
                add("rows_conv", "fp32", items * (2 * 5.0 * n * l2 + 16.0 * n))
        elif t == mg.NodeType.EQ:
            big = slots * batch * -(-length // 6144) >= nsm  # eq.cu eq_uses_small_window
            nw, hop = (8192, 6144) if big else (4096, 2048)
            wins = slots * batch * -(-length // hop)
            add("eq_conv", "fp32", wins * (2 * 5.0 * nw * (13 if big else 12) + 8.0 * nw))
        elif t in fam_of:
            add("dyn_scan", "hbm", hbm)
        elif t != mg.NodeType.IN:
            add("pointwise", "hbm", hbm)
    return out


def roofline_table(fam_serial, work, hbm_peak):
    """Per kernel family: serialized in-render time, algorithmic work, achieved and fraction of
    its bound's peak (nominal FP32 for FFT families, measured HBM for the others). An HBM family
    can exceed 1.0: rows written by the step just before it are partly still in L2 (the master
    mix reads the reverb / delay outputs the previous steps just stored)."""
    tab, merged = {}, {}
    for k, d in fam_serial.items():  # pointwise / pointwise_wide / pointwise_chain: one family
        m = merged.setdefault("pointwise" if k.startswith("pointwise") else k, {"us": 0.0, "launches": 0})
        m["us"] += d["us"]
        m["launches"] += d["launches"]
    for k, d in merged.items():
        row = {"us": round(d["us"], 1), "launches": d["launches"]}
        if k in work and d["us"] > 0:
            bound, w = work[k]
            if bound == "fp32":
                a = w / (d["us"] * 1e-6) / 1e12
                row.update(bound="fp32", flops=w, achieved_tflops=round(a, 3), frac=round(a / FP32_PEAK_TFLOPS, 4))
            else:
                a = w / (d["us"] * 1e-6) / 1e9
                row.update(bound="hbm", bytes=w, achieved_gbs=round(a, 1), frac=round(a / hbm_peak, 4))
        tab[k] = row
    return dict(sorted(tab.items(), key=lambda kv: -kv[1]["us"]))


# ---- reference CPU renders (cpu_baseline and --impl reference) -----------------------------

def _ref_render_graphs(args):
    idx, reps = args
    from oracle import ref
    graphs = wl.config5_graphs()
    bank = wl.source_bank(64, L)
    ns, dt = 0, 0.0
    for _ in range(reps):
        for i in idx:
            t, e = graphs[i]
            k = int(np.sum(t == 0))
            src = bank[[j % 64 for j in range(k)]]
            p = ref.Plan(t, e, 1)
            t0 = time.perf_counter()
            p.render(wl.config5_member_params(i, t), src, sample_rate=FS)
            dt += time.perf_counter() - t0
            ns += node_samples(t)
    return ns, dt


def reference_sample(procs_n, graphs_per_proc, step):
    """One bounded step of the reference on `procs_n` processes: graphs step*P*G + ... of the
    512-graph set (a rotating sample); returns (node-samples, wall seconds)."""
    import multiprocessing as mp
    start = (step * procs_n * graphs_per_proc) % 512
    work = [([(start + p * graphs_per_proc + j) % 512 for j in range(graphs_per_proc)], 1) for p in range(procs_n)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs_n) as pool:
        t0 = time.perf_counter()
        res = pool.map(_ref_render_graphs, work)
        wall = time.perf_counter() - t0
    return sum(r[0] for r in res), wall


def reference_arm(args):
    rank, world, _ = dist_setup()
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmixgraph_ref.so not built"}))
        return
    cores = os.cpu_count() or 1
    warm = max(1, min(args.warmup, 1))
    steps = max(1, min(args.steps, 12))
    for s in range(warm):
        reference_sample(cores, 1, s)
    ns, wall = 0, 0.0
    for s in range(steps):
        n, w = reference_sample(cores, 1, warm + s)
        ns, wall = ns + n, wall + w
    value = ns / wall
    sample = (f"{steps} steps x {cores} processes x 1 config-5 graph each (rotating through the 512-graph set; "
              f"reference render(), oracle/_ref with the FFTW-API stand-in FFT), {wall:.1f} s wall")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "graph_renders_per_sec": steps * cores / wall, "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": wall / steps * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generators: generate_console, random_legal_params, uniform_noise)",
        "config": {"workload": WORKLOAD, "length": L, "batch": 1, "sample_rate": FS},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ---- secondary configs (N = 1) ---------------------------------------------------------------

def config2_lines(mg, procs, dev, steps=20, warmup=3):
    """Config 2 (console-16, 121 nodes, 2^17): device time of the captured render (L2 flushed
    between iterations) and e2e through RenderPipeline with double host audio."""
    import torch
    t, e, params = wl.config2()
    rd = mg.compute_render_data_arrays(t, e)
    P = rd.reorder_params(params)
    src = wl.sources(rd.num_inputs, L)
    dr = mg.DeviceRenderer(rd, procs, 1, L, P, device=dev)
    dr.sources.copy_(torch.as_tensor(src, dtype=torch.float32))
    g = dr.capture()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        g.replay()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        g.replay()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    ns = node_samples(t)
    fam, span = in_render_kernel_times(g.replay)
    dr.render_profiled(hoist=False)
    fam_s, span_s = in_render_kernel_times(lambda: dr.render_profiled(hoist=False))
    serial = roofline_table(fam_s, family_work(mg, procs, rd, L), peaks()[0])
    pipe = mg.RenderPipeline(rd, procs, 1, L, dtype=np.float64, depth=2)
    ps = pipe.pinned(src.shape)
    ps[...] = src
    outs = [pipe.pinned((rd.buffer_rows - rd.output_begin, 1, 2, L)) for _ in range(2)]
    for i in range(3):
        pipe.submit(P, ps, outs[i % 2])
    pipe.sync()
    t0 = time.perf_counter()
    for i in range(steps):
        pipe.submit(P, ps, outs[i % 2])
    pipe.sync()
    e2e_s = (time.perf_counter() - t0) / steps
    del g, dr, pipe, flush
    torch.cuda.empty_cache()
    return {"value": ns / (ms * 1e-3), "unit": UNIT, "ms_per_render": ms, "graph_renders_per_sec": 1e3 / ms,
            "e2e": {"value": ns / e2e_s, "unit": UNIT, "ms_per_render": e2e_s * 1e3,
                    "api": "RenderPipeline (mg_pipeline_submit), double host audio, pinned"},
            "in_render_us": {k: round(v["us"], 1) for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["us"])},
            "render_span_us_traced": span, "roofline_families_serialized": serial,
            "serialized_span_us": span_s, "gpu_launches_per_render": rd.kernel_count(1, L),
            "workload": "config2: generate_console(16, p=0.3, seed=16), 121 nodes / 139 edges, stereo 2^17, B=1; "
                        "L2 flushed between iterations",
            "type_string": rd.schedule.type_codes()}


def config3_rate(mg, procs, dev, steps=6, warmup=2, graphs=64):
    """Config 3: 64 consoles per step with topology re-drawn every step (wl.config3_members);
    plan build (compute_render_data, C++) on a worker thread one batch ahead, then
    BatchRenderer.submit (async plan + original-order parameter upload, device reorder,
    render, 64-output D2H). Wall clock over the timed steps, host plan build included."""
    import queue

    import torch

    from paper_2408_03204_b200 import sharding
    batches = []
    for st in range(warmup + steps):
        members = wl.config3_members(st, graphs)
        t, e = sharding.union_arrays(members)
        batches.append((t, e, wl.random_legal_params(t, wl.config3_params_seed(st))))
    cap = np.zeros(4, dtype=np.uint64)
    for t, e, _ in batches:
        cap = np.maximum(cap, mg.BatchRenderer.capacity_of(mg.compute_render_data_arrays(t, e), procs, 1, L))
    br = mg.BatchRenderer(procs, 1, L, cap, depth=2)
    bank = torch.as_tensor(wl.source_bank(64, L), dtype=torch.float32).to(dev)
    outs = [torch.empty((graphs, 1, 2, L), dtype=torch.float32, pin_memory=True).numpy() for _ in range(2)]
    q = queue.Queue(maxsize=2)

    def producer():
        for t, e, params in batches:
            q.put((mg.compute_render_data_arrays(t, e), params, t))

    th = threading.Thread(target=producer, daemon=True)
    th.start()
    ns, t0 = 0, None
    for i in range(warmup + steps):
        rd, params, t = q.get()
        if i == warmup:
            br.sync()
            t0 = time.perf_counter()
        br.submit(rd, params, bank, outs[i % 2], validate=True)
        if i >= warmup:
            ns += node_samples(t)
    br.sync()
    dt = time.perf_counter() - t0
    th.join()
    del br, bank
    torch.cuda.empty_cache()
    return {"value": ns / dt, "unit": UNIT, "graph_renders_per_sec": graphs * steps / dt, "steps": steps,
            "warmup": warmup, "ms_per_step": dt / steps * 1e3, "graphs_per_step": graphs,
            "workload": "config3: 64 random consoles per step (K in [4,32], p=0.3), topology re-drawn every step, "
                        "stereo 2^17; plan build one batch ahead on a worker thread; BatchRenderer; wall clock",
            "data": "synthetic; sources from a 64-row device noise bank"}


def config4_rate(mg, procs, dev, steps=3, warmup=2):
    """Config 4: generate_large_console(64), 966 nodes, 10 s (L = 441,000; the reverb/delay
    convolutions as three 2^18-point overlap-save segments): forward (captured render) and the
    optimisation step (forward + MSE + reverse-mode pass over every parameter + update).
    Device time (CUDA events)."""
    import torch

    from paper_2408_03204_b200 import training
    L4 = wl.L4
    t, e = wl.generate_large_console_arrays(64)
    rd = mg.compute_render_data_arrays(t, e)
    P = rd.reorder_params(wl.random_legal_params(t, 4040))
    tr = training.Trainer(rd, procs, 1, L4, P, trainable=[int(x) for x in P], learning_rate=1e-3, device=dev)
    src = torch.as_tensor(wl.sources(rd.num_inputs, L4), dtype=torch.float32).to(dev)
    tgt = torch.zeros((rd.buffer_rows - rd.output_begin, 1, 2, L4), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    tr.dr.sources.copy_(src)
    graph = tr.dr.capture()

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in ev:
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev) / steps

    fwd_ms = timed(graph.replay)
    train_ms = timed(lambda: tr.step(src, tgt))
    ns = node_samples(t, L4)
    out = {"value": ns / (train_ms * 1e-3), "unit": UNIT, "graph_renders_per_sec": 1e3 / train_ms,
           "ms_per_step": train_ms, "forward_ms": fwd_ms, "forward_node_samples_per_sec": ns / (fwd_ms * 1e-3),
           "steps": steps, "warmup": warmup, "nodes": len(t), "edges": len(e), "type_string": rd.schedule.type_codes(),
           "workload": "config4: generate_large_console(64), 966 nodes / 1093 edges, stereo 10 s (L=441000) @ "
                       "44.1 kHz, B=1; step = forward + MSE + backward (all parameter gradients) + SGD update",
           "data": "synthetic (uniform_noise sources, random_legal_params, zero target)"}
    del graph, tr
    torch.cuda.empty_cache()
    return out


def config5_train_rate(mg, procs, dev, rank, world, steps=4, warmup=2, batch=2):
    """Config 5's optimisation variant: one console-16 parameter set shared by every rank,
    each rank a batch of its own sources (data parallel); step = forward + MSE + backward +
    ONE all-reduce of the flat fp64 gradient buffer + gradient step. Weak scaling."""
    import torch
    import torch.distributed as dist

    from paper_2408_03204_b200 import training
    t, e, params = wl.config2()
    rd = mg.compute_render_data_arrays(t, e)
    P = rd.reorder_params(wl.random_legal_params(t, 2024))
    tr = training.Trainer(rd, procs, batch, L, P, trainable=[int(x) for x in P], learning_rate=1e-3,
                          group=dist.group.WORLD if world > 1 else None, device=dev)
    src = torch.as_tensor(wl.sources(rd.num_inputs, L, batch, base_seed=1000 + 100 * rank), dtype=torch.float32).to(dev)
    tgt = torch.zeros((rd.buffer_rows - rd.output_begin, batch, 2, L), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        tr.step(src, tgt)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        tr.step(src, tgt)
    b.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / steps, dev, world)
    ns = node_samples(t) * batch * world
    grad_bytes = int(tr.flat.numel() * 8)
    del tr
    torch.cuda.empty_cache()
    return {"value": ns / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps, "warmup": warmup,
            "n_gpus": world, "scaling": "weak", "batch_per_rank": batch, "allreduce_bytes": grad_bytes,
            "collective": "all-reduce (sum) of the flat fp64 gradient buffer, 1 per step" if world > 1 else "none (1 GPU)",
            "workload": "config5 optimisation: console-16 (121 nodes) shared parameters, per-rank batch of 2 stereo "
                        "2^17 sources; forward + MSE + backward + all-reduce + SGD (all types trainable)",
            "data": "synthetic (uniform_noise sources, zero target)"}


_BACKEND = "nccl"


def max_over_ranks(x, dev, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev if _BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---- the B200 arm ---------------------------------------------------------------------------

def b200_arm(args):
    global _BACKEND
    import torch
    import torch.distributed as dist

    import paper_2408_03204_b200 as mg

    rank, world, local = dist_setup()
    ndev = max(1, torch.cuda.device_count())
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    _BACKEND = args.backend
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    procs = mg.ProcessorSet(sample_rate=FS, device=dev_index)
    graphs, mine, unions = config5_shard(rank, world)
    ns_all = sum(node_samples(t) for t, _ in graphs)
    ns_mine = sum(node_samples(graphs[i][0]) for i in mine)
    bank_host = wl.source_bank(64, L)
    bank = torch.as_tensor(bank_host, dtype=torch.float32).to(dev)

    # Device-resident renders: one DeviceRenderer + captured graph per union, inputs copied in
    # once (input k <- bank row k % 64).
    cases, renderers, captured, kernels_per_step = [], [], [], 0
    for idx in unions:
        t, rd, params = union_case(mg, graphs, idx)
        dr = mg.DeviceRenderer(rd, procs, 1, L, rd.reorder_params(params), device=dev)
        dr.sources.copy_(bank[torch.arange(rd.num_inputs, device=dev) % 64])
        renderers.append(dr)
        captured.append(dr.capture())
        cases.append((t, rd, params))
        kernels_per_step += rd.kernel_count(1, L)
    stream = torch.cuda.current_stream(dev)

    def step():
        for g in captured:
            g.replay()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    n = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    sampler = ClockSampler(dev_index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    wall0 = time.perf_counter()
    for i in range(n):
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    dev_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    dev_ms_max = max_over_ranks(dev_ms, dev, world)

    # In-render kernel timings of one step (CUPTI traces, outside the timed region): the
    # replayed step as timed (concurrent kernels overlap, low-priority prologues include time
    # waiting for SMs) and the same renders serialised on one stream (each kernel's own cost,
    # with the render's cache state) for the roofline.
    fam, span_us = in_render_kernel_times(step)

    def serial_step():
        for dr in renderers:
            dr.render_profiled(hoist=False)

    serial_step()
    fam_serial, serial_span_us = in_render_kernel_times(serial_step)
    work = {}
    for _, rd, _ in cases:
        for k, (bound, w) in family_work(mg, procs, rd, L).items():
            work[k] = (bound, work.get(k, (bound, 0.0))[1] + w)

    # End to end through the public API with host buffers: BatchRenderer (mg_batch_submit),
    # pinned fp32 sources per input node, original-order parameters, outputs D2H.
    cap = np.zeros(4, dtype=np.uint64)
    for _, rd, _ in cases:
        cap = np.maximum(cap, mg.BatchRenderer.capacity_of(rd, procs, 1, L))
    for dr in renderers:
        del dr
    del captured, renderers
    torch.cuda.empty_cache()
    br = mg.BatchRenderer(procs, 1, L, cap, depth=2)
    src_pin = torch.empty(bank_host.shape, dtype=torch.float32, pin_memory=True).numpy()
    src_pin[...] = bank_host
    outs = [torch.empty((rd.buffer_rows - rd.output_begin, 1, 2, L), dtype=torch.float32, pin_memory=True).numpy()
            for _, rd, _ in cases]
    row_bytes = 4 * 2 * L
    h2d = sum(rd.num_inputs * row_bytes + int(sum(v.size for v in p.values())) * 8 for _, rd, p in cases)
    d2h = sum(o.nbytes for o in outs)

    def e2e_step():
        for (_, rd, params), o in zip(cases, outs):
            br.submit(rd, params, src_pin, o, validate=False)
        br.sync()

    for _ in range(2):
        e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n):
        e2e_step()
    e2e_s = max_over_ranks(time.perf_counter() - t0, dev, world)
    del br
    torch.cuda.empty_cache()

    extras = {}
    if not args.no_extras:
        try:
            extras["config5_train"] = config5_train_rate(mg, procs, dev, rank, world)
        except Exception as ex:  # report, never lose the headline line
            extras["config5_train"] = {"error": repr(ex)[:300]}
        if world == 1:
            for key, fn in (("config2", config2_lines), ("config3", config3_rate), ("config4", config4_rate)):
                try:
                    extras[key] = fn(mg, procs, dev)
                except Exception as ex:
                    extras[key] = {"error": repr(ex)[:300]}

    alg_bytes = sum(8.0 * L * (len(st.gather) + st.store_end - st.store_begin) for _, rd, _ in cases for st in rd.steps)
    if rank == 0:
        hbm_peak, peak_kind = peaks()
        value = ns_all * n / (dev_ms_max * 1e-3)
        # Dominant kernel family by its serialised in-render time, and its roofline.
        table = roofline_table(fam_serial, work, hbm_peak)
        dom_name = next(iter(table)) if table else None
        dom = table.get(dom_name, {})
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "r02s_traffic.json")) as f:
                traffic = (json.load(f).get(dom_name) or {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        result = {
            "metric": METRIC, "value": value, "unit": UNIT,
            "graph_renders_per_sec": len(graphs) * n / (dev_ms_max * 1e-3),
            "n_gpus": world, "steps": n, "warmup": max(args.warmup, 3), "ms_per_step": dev_ms_max / n,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generators: generate_console, random_legal_params, uniform_noise bank)",
            "config": {"workload": WORKLOAD, "graphs": len(graphs), "graphs_on_rank0": len(mine), "unions_on_rank0": len(unions),
                       "length": L, "batch": 1, "sample_rate": FS, "node_samples_per_step": ns_all,
                       "l2": "inputs larger than L2 (each union's arena is ~8 GB), no flush",
                       "parallelism": f"graph-sharded x{world} ({args.backend})",
                       "execution": "per-union CUDA graph replay; parameter-only prologues on side streams"},
            "e2e": {"value": ns_all * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "BatchRenderer (mg_batch_submit): pinned fp32 host sources per input node, original-order "
                           "parameter tables, device reorder, render, output D2H; wall clock, max over ranks",
                    "ms_per_step": e2e_s / n * 1e3, "graph_renders_per_sec": len(graphs) * n / e2e_s},
            "roofline": {"bound": dom.get("bound"), "kernel": dom_name,
                         "achieved": dom.get("achieved_tflops", dom.get("achieved_gbs")),
                         "peak": FP32_PEAK_TFLOPS if dom.get("bound") == "fp32" else hbm_peak,
                         "peak_kind": ("nominal FP32 CUDA-core (148 SM x 128 FMA x 2 x 1965 MHz); no measured FP32 "
                                       "peak" if dom.get("bound") == "fp32" else peak_kind),
                         "unit": "TFLOP/s" if dom.get("bound") == "fp32" else "GB/s", "frac": dom.get("frac"),
                         "traffic": traffic, "launches_per_step": dom.get("launches"),
                         "us_per_step_serialized": dom.get("us"),
                         "work_per_step": dom.get("flops", dom.get("bytes")),
                         "share_of_serialized_kernel_time": (dom.get("us", 0.0) / sum(v["us"] for v in table.values())
                                                             if table else None),
                         "note": "dominant kernel family by in-render time with the step's renders serialised on one "
                                 "stream (CUPTI trace, prologues inline, no side streams: each kernel's own cost "
                                 "with the render's cache state); work = algorithmic flops of the implemented "
                                 "transforms (5 N log2 N per complex N-point transform + 8 per spectral product) "
                                 "or algorithmic bytes; traffic = ncu dram bytes per launch of that family from "
                                 "the committed capture (profiles/r02s_traffic.json)"},
            "roofline_families": table,
            "roofline_hbm": {"bound": "hbm", "achieved": alg_bytes / (dev_ms / n * 1e-3) / 1e9,
                             "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s", "traffic": alg_bytes,
                             "note": "whole render of rank 0's shard: algorithmic bytes (every gathered row read once, "
                                     "every non-input row written once, 8 B per stereo sample) over the device step "
                                     "time; SURVEY.md 8d"},
            "in_render_us_per_step": {k: round(v["us"], 1) for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["us"])},
            "serialized_span_us": serial_span_us,
            "in_render_launches_per_step": {k: v["launches"] for k, v in fam.items()},
            "traced_span_us": span_us,
            "wall_s_timed_region": wall, "clocks": clocks, "gpu_launches": kernels_per_step * n,
        }
        result["roofline_hbm"]["frac"] = result["roofline_hbm"]["achieved"] / hbm_peak
        result.update(extras)
        if world == 1 and not args.no_cpu_baseline:
            try:
                from oracle import ref
                if ref.available():
                    cores = os.cpu_count() or 1
                    nsr, w = reference_sample(cores, 1, 0)
                    result["cpu_baseline"] = {
                        "value": nsr / w, "unit": UNIT, "cores": cores, "kind": "reference",
                        "sample": f"{cores} config-5 graphs, one per host process (reference render(), oracle/_ref, "
                                  f"FFTW-API stand-in FFT), {w:.1f} s wall"}
            except Exception as ex:
                result["cpu_baseline"] = {"error": repr(ex)[:200]}
        print(json.dumps(result))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
