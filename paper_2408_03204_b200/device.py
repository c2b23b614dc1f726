"""Device-resident render path: one fp32 HBM arena per (plan, batch, length).

Wraps ``mg_render_arena`` (include/mixgraph_b200.h). torch is used only for device memory,
streams and events (plumbing); all arithmetic runs in the library's sm_100a kernels.

Arena layout: ``arena[row, b, c, n]`` with rows in render (reordered) order; rows
``[0, num_inputs)`` are the sources, rows ``[output_begin, buffer_rows)`` the outputs
(`render.cpp:32-37,63-69`). Parameter tables live on the device in fp64, render order.
"""
from __future__ import annotations

import ctypes
from typing import Dict, Optional

import numpy as np
import torch

from . import NUM_NODE_TYPES, ProcessorSet, RenderData, _check, _lib, _u64, _vp, param_width


class DeviceRenderer:
    def __init__(self, rd: RenderData, procs: ProcessorSet, batch: int, length: int,
                 params: Optional[Dict[int, np.ndarray]] = None, device: Optional[torch.device] = None,
                 arena_pool: Optional[torch.Tensor] = None, workspace_pool: Optional[torch.Tensor] = None,
                 backward: bool = False):
        """`arena_pool` (fp32) / `workspace_pool` (uint8): optional preallocated device buffers
        at least as large as this plan needs, reused across plans whose topology changes every
        step (no per-plan allocation). The arena view is NOT zeroed in that case.
        `backward`: size the workspace for backward() after render()."""
        if not torch.cuda.is_available():
            raise RuntimeError("DeviceRenderer needs a CUDA device (there is no CPU fallback)")
        self.rd, self.procs = rd, procs
        self.batch, self.length = int(batch), int(length)
        self.device = device or torch.device("cuda", procs.device)
        shape = (rd.buffer_rows, self.batch, 2, self.length)
        if arena_pool is None:
            self.arena = torch.zeros(shape, dtype=torch.float32, device=self.device)
        else:
            need = rd.buffer_rows * self.batch * 2 * self.length
            if arena_pool.dtype != torch.float32 or arena_pool.numel() < need:
                raise ValueError(f"DeviceRenderer: arena_pool must be float32 with >= {need} elements")
            self.arena = arena_pool.reshape(-1)[:need].view(shape)
        ws = _u64()
        fn = _lib.mg_backward_workspace_bytes if backward else _lib.mg_plan_workspace_bytes
        _check(fn(rd.handle, procs.handle, self.batch, self.length, ctypes.byref(ws)))
        self.adjoint: Optional[torch.Tensor] = None
        self.workspace_bytes = int(ws.value)
        if workspace_pool is None:
            self.workspace = torch.empty(self.workspace_bytes, dtype=torch.uint8, device=self.device)
        else:
            if workspace_pool.dtype != torch.uint8 or workspace_pool.numel() < self.workspace_bytes:
                raise ValueError(f"DeviceRenderer: workspace_pool must be uint8 with >= {self.workspace_bytes} bytes")
            self.workspace = workspace_pool.reshape(-1)[:self.workspace_bytes]
        self.tables: Dict[int, torch.Tensor] = {}
        self._ptrs = (_vp * NUM_NODE_TYPES)()
        self.set_params(rd.flat.params if params is None else params)

    def set_params(self, params: Dict[int, np.ndarray]) -> None:
        """Upload render-order parameter tables (RenderData.reorder_params layout).

        After the first upload the tables are rewritten IN PLACE: a captured RenderGraph bakes
        their device addresses, so a new set must have the same types and shapes (ValueError
        otherwise; build a new DeviceRenderer for a different table set)."""
        new = {int(t): torch.as_tensor(np.ascontiguousarray(m, dtype=np.float64).reshape(-1, param_width(int(t))))
               for t, m in params.items()}
        if self.tables:
            if set(new) != set(self.tables) or any(new[t].shape != self.tables[t].shape for t in new):
                raise ValueError("DeviceRenderer.set_params: parameter tables must keep their types and shapes "
                                 "(captured render graphs hold their addresses)")
            for t, a in new.items():
                self.tables[t].copy_(a)
            return
        for t in range(NUM_NODE_TYPES):
            self._ptrs[t] = None
        for t, a in new.items():
            d = a.to(self.device)
            self.tables[t] = d
            self._ptrs[t] = d.data_ptr()

    @property
    def sources(self) -> torch.Tensor:
        return self.arena[: self.rd.num_inputs]

    @property
    def outputs(self) -> torch.Tensor:
        return self.arena[self.rd.output_begin:]

    def kernel_count(self) -> int:
        return self.rd.kernel_count(self.batch, self.length)

    def render(self, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Enqueue every render step on `stream` (default: torch's current stream)."""
        s = stream or torch.cuda.current_stream(self.device)
        _check(_lib.mg_render_arena(self.rd.handle, self.procs.handle, self._ptrs,
                                    ctypes.c_void_p(self.arena.data_ptr()), self.batch, self.length,
                                    ctypes.c_void_p(self.workspace.data_ptr()), self.workspace_bytes,
                                    ctypes.c_void_p(s.cuda_stream)))
        return self.outputs

    def backward(self, grad_outputs: torch.Tensor, stream: Optional[torch.cuda.Stream] = None,
                 grads: Optional[Dict[int, torch.Tensor]] = None):
        """Reverse-mode pass after render() (mg_render_backward_arena): `grad_outputs`
        [num_outputs][batch][2][length] = dL/d(outputs). Returns (grads, grad_sources): grads
        per type, device fp64 in render order (rd.original_order maps them back), and
        dL/d(sources) [num_inputs][batch][2][length] fp32 (a view into the adjoint arena).
        Needs DeviceRenderer(..., backward=True). `grads`: optional preallocated output tables
        (fp64, shaped like the parameter tables, e.g. views into one flat all-reduce buffer)."""
        s = stream or torch.cuda.current_stream(self.device)
        if self.adjoint is None:
            self.adjoint = torch.empty_like(self.arena)
        self.adjoint[self.rd.output_begin:].copy_(grad_outputs)
        if grads is None:
            grads = {t: torch.empty_like(tab) for t, tab in self.tables.items()}
        gptrs = (_vp * NUM_NODE_TYPES)()
        for t, tab in self.tables.items():
            g = grads[t]
            if g.dtype != torch.float64 or g.shape != tab.shape or not g.is_contiguous():
                raise ValueError("backward: gradient tables must be contiguous fp64 shaped like the parameters")
            gptrs[t] = g.data_ptr()
        with torch.cuda.stream(s):
            _check(_lib.mg_render_backward_arena(self.rd.handle, self.procs.handle, self._ptrs,
                                                 ctypes.c_void_p(self.arena.data_ptr()),
                                                 ctypes.c_void_p(self.adjoint.data_ptr()), gptrs, self.batch,
                                                 self.length, ctypes.c_void_p(self.workspace.data_ptr()),
                                                 self.workspace_bytes, ctypes.c_void_p(s.cuda_stream)))
        return grads, self.adjoint[: self.rd.num_inputs]

    def capture(self) -> "RenderGraph":
        """Capture one full render (main stream + side-stream prologues) as a CUDA graph
        instantiated with node priorities (mg_render_graph_create); replay() re-runs it on
        the current arena, parameter tables and workspace (contents may change in place)."""
        return RenderGraph(self)

    def render_profiled(self, stream: Optional[torch.cuda.Stream] = None, sync: bool = False,
                        hoist: bool = True) -> Optional[np.ndarray]:
        """Same as render() with CUDA events around every step on the launching stream. With
        sync=True, waits and returns per-step device times (ms, one per RenderData step);
        hoist=False runs each step's parameter prologue inline (isolated per-step costs)."""
        s = stream or torch.cuda.current_stream(self.device)
        out = np.zeros(self.rd.num_steps, dtype=np.float32) if sync else None
        _check(_lib.mg_render_arena_profiled(self.rd.handle, self.procs.handle, self._ptrs,
                                             ctypes.c_void_p(self.arena.data_ptr()), self.batch, self.length,
                                             ctypes.c_void_p(self.workspace.data_ptr()), self.workspace_bytes,
                                             ctypes.c_void_p(s.cuda_stream),
                                             None if out is None else out.ctypes.data_as(ctypes.c_void_p),
                                             int(hoist)))
        return out


def profile_steps(dr: "DeviceRenderer", reps: int = 20, stream: Optional[torch.cuda.Stream] = None) -> np.ndarray:
    """Per-step device time in ms (prologue + audio pass of each RenderData step), each step
    repeated `reps` times back to back between one CUDA event pair (mg_profile_steps)."""
    s = stream or torch.cuda.current_stream(dr.device)
    out = np.zeros(dr.rd.num_steps, dtype=np.float32)
    _check(_lib.mg_profile_steps(dr.rd.handle, dr.procs.handle, dr._ptrs, ctypes.c_void_p(dr.arena.data_ptr()),
                                 dr.batch, dr.length, ctypes.c_void_p(dr.workspace.data_ptr()), dr.workspace_bytes,
                                 ctypes.c_void_p(s.cuda_stream), int(reps), out.ctypes.data_as(ctypes.c_void_p)))
    return out


class RenderGraph:
    def __init__(self, dr: DeviceRenderer):
        self._dr = dr  # keeps the arena / workspace / tables alive
        self._h = ctypes.c_void_p()
        _check(_lib.mg_render_graph_create(dr.rd.handle, dr.procs.handle, dr._ptrs,
                                           ctypes.c_void_p(dr.arena.data_ptr()), dr.batch, dr.length,
                                           ctypes.c_void_p(dr.workspace.data_ptr()), dr.workspace_bytes,
                                           ctypes.byref(self._h)))

    def replay(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream or torch.cuda.current_stream(self._dr.device)
        _check(_lib.mg_render_graph_launch(self._h, ctypes.c_void_p(s.cuda_stream)))

    def __del__(self, _destroy=_lib.mg_render_graph_destroy):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _destroy(h)


class RenderPipeline:
    """Streaming host-buffer renders (mg_pipeline_*): submit() returns immediately; the H2D
    copies of render i+1 overlap the kernels of render i. `dtype` is the host audio type
    (np.float32: copied straight into the arena; np.float64: reference AudioBuffer precision,
    converted to fp32 on host worker threads in 1 MiB chunks whose H2D copies start as each
    chunk is done — half the PCIe bytes; host_threads=0 sends double and converts on the
    device instead; -1 picks from the host's core count and LOCAL_WORLD_SIZE). Host arrays should be pinned (see `pinned`) and must stay alive
    until sync() — the pipeline keeps references until then."""

    def __init__(self, rd: RenderData, procs: ProcessorSet, batch: int, length: int, dtype=np.float32, depth: int = 2,
                 host_threads: int = -1):
        from . import _tables  # noqa: F401
        self.rd, self.procs = rd, procs
        self.batch, self.length = int(batch), int(length)
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise ValueError("RenderPipeline: dtype must be float32 or float64")
        self._h = ctypes.c_void_p()
        _check(_lib.mg_pipeline_create(rd.handle, procs.handle, self.batch, self.length,
                                       int(self.dtype == np.float32), int(depth), int(host_threads),
                                       ctypes.byref(self._h)))
        self._keep = []

    def pinned(self, shape) -> np.ndarray:
        """A page-locked host array of this pipeline's dtype."""
        tdt = torch.float32 if self.dtype == np.float32 else torch.float64
        t = torch.empty(tuple(shape), dtype=tdt, pin_memory=True)
        arr = t.numpy()
        self._keep.append(t)
        return arr

    def submit(self, params: Dict[int, np.ndarray], sources: np.ndarray, out: np.ndarray) -> None:
        from . import _tables
        k = self.rd.num_inputs
        o = self.rd.buffer_rows - self.rd.output_begin
        want_s = (k, self.batch, 2, self.length)
        want_o = (o, self.batch, 2, self.length)
        for a, shape in ((sources, want_s), (out, want_o)):
            if a.shape != shape:
                raise ValueError(f"RenderPipeline: expected {shape}, got {a.shape}")
            if a.dtype != self.dtype or not a.flags.c_contiguous:
                raise ValueError(f"RenderPipeline: arrays must be contiguous {self.dtype}")
        ptrs, rows, keep = _tables(params)
        _check(_lib.mg_pipeline_submit(self._h, ptrs, rows.ctypes.data_as(_vp),
                                       ctypes.c_void_p(sources.ctypes.data), ctypes.c_void_p(out.ctypes.data)))
        self._keep.append((sources, out))

    def sync(self) -> None:
        _check(_lib.mg_pipeline_sync(self._h))
        self._keep = [x for x in self._keep if isinstance(x, torch.Tensor)]

    def __del__(self, _destroy=_lib.mg_pipeline_destroy):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _destroy(h)


class BatchRenderer:
    """Renders of plans whose topology changes every batch (mg_batch_*, BASELINE config 3).

    Device pools are sized once (`capacity`: [arena rows, workspace bytes, step-table ints,
    parameter doubles], e.g. the max of `BatchRenderer.capacity_of(rd, ...)` over a dataset);
    submit() packs the plan's step table and the ORIGINAL-order parameter tables into pinned
    staging, uploads them on a copy stream, reorders the parameters on the device and enqueues
    the render, without allocating or synchronising — the host prepares batch i+1 while the
    GPU renders batch i. Plans and host arrays are kept alive until their slot is reused."""

    def __init__(self, procs: ProcessorSet, batch: int, length: int, capacity, depth: int = 2):
        self.procs, self.batch, self.length, self.depth = procs, int(batch), int(length), int(depth)
        cap = np.ascontiguousarray(np.asarray(capacity, dtype=np.uint64).reshape(4))
        self.capacity = cap
        self._h = ctypes.c_void_p()
        _check(_lib.mg_batch_create(procs.handle, self.batch, self.length, cap.ctypes.data_as(_vp), self.depth,
                                    ctypes.byref(self._h)))
        self._keep = [None] * self.depth
        self._n = 0

    @staticmethod
    def capacity_of(rd: RenderData, procs: ProcessorSet, batch: int, length: int) -> np.ndarray:
        cap = np.zeros(4, dtype=np.uint64)
        _check(_lib.mg_batch_capacity(rd.handle, procs.handle, int(batch), int(length), cap.ctypes.data_as(_vp)))
        return cap

    def submit(self, rd: RenderData, params: Dict[int, np.ndarray], sources, outputs: Optional[np.ndarray] = None,
               validate: bool = True) -> None:
        """`params`: per-type tables in ORIGINAL row order; `sources`: float32
        [rows][batch][2][length] torch CUDA tensor (device) or numpy array (host, ideally
        pinned); input k of the plan takes source row k % rows. `outputs`: optional host
        float32 [num_outputs][batch][2][length] array filled asynchronously (valid after sync)."""
        from . import _tables
        ptrs, rows, keep = _tables(params)
        if isinstance(sources, torch.Tensor):
            if not sources.is_cuda or sources.dtype != torch.float32 or not sources.is_contiguous():
                raise ValueError("BatchRenderer: device sources must be a contiguous float32 CUDA tensor")
            src_ptr, src_rows, on_dev = sources.data_ptr(), int(sources.shape[0]), 1
            row = sources[0].numel()
        else:
            if sources.dtype != np.float32 or not sources.flags.c_contiguous:
                raise ValueError("BatchRenderer: host sources must be contiguous float32")
            src_ptr, src_rows, on_dev = sources.ctypes.data, int(sources.shape[0]), 0
            row = sources[0].size
        if row != self.batch * 2 * self.length:
            raise ValueError(f"BatchRenderer: source rows must be [{self.batch}][2][{self.length}]")
        out_ptr = None
        if outputs is not None:
            want = (rd.buffer_rows - rd.output_begin, self.batch, 2, self.length)
            if outputs.shape != want or outputs.dtype != np.float32 or not outputs.flags.c_contiguous:
                raise ValueError(f"BatchRenderer: outputs must be contiguous float32 {want}")
            out_ptr = outputs.ctypes.data
        _check(_lib.mg_batch_submit(self._h, rd.handle, ptrs, rows.ctypes.data_as(_vp), int(bool(validate)),
                                    ctypes.c_void_p(src_ptr), src_rows, on_dev, out_ptr))
        self._keep[self._n % self.depth] = (rd, keep, sources, outputs)
        self._n += 1

    def sync(self) -> None:
        _check(_lib.mg_batch_sync(self._h))

    def last_outputs(self) -> torch.Tensor:
        """Device view of the most recent submit's output rows (valid after sync)."""
        rd = self._keep[(self._n - 1) % self.depth][0]
        p = ctypes.c_void_p()
        _check(_lib.mg_batch_last_arena(self._h, ctypes.byref(p)))
        n = rd.buffer_rows * self.batch * 2 * self.length
        arena = _device_view(p.value, n, self.procs.device).view(rd.buffer_rows, self.batch, 2, self.length)
        return arena[rd.output_begin:]

    def __del__(self, _destroy=_lib.mg_batch_destroy):
        h, self._h = getattr(self, "_h", None), None
        if h:
            _destroy(h)


def _device_view(ptr: int, n: int, device: int) -> torch.Tensor:
    """A float32 torch view of `n` elements of library-owned device memory (no copy)."""
    class _Iface:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3, "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Iface(), device=f"cuda:{device}")
