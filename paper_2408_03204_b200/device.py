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
                 arena_pool: Optional[torch.Tensor] = None, workspace_pool: Optional[torch.Tensor] = None):
        """`arena_pool` (fp32) / `workspace_pool` (uint8): optional preallocated device buffers
        at least as large as this plan needs, reused across plans whose topology changes every
        step (no per-plan allocation). The arena view is NOT zeroed in that case."""
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
        _check(_lib.mg_plan_workspace_bytes(rd.handle, procs.handle, self.batch, self.length, ctypes.byref(ws)))
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
        """Upload render-order parameter tables (RenderData.reorder_params layout)."""
        self.tables = {}
        for t in range(NUM_NODE_TYPES):
            self._ptrs[t] = None
        for t, m in params.items():
            a = torch.as_tensor(np.ascontiguousarray(m, dtype=np.float64).reshape(-1, param_width(t)))
            d = a.to(self.device)
            self.tables[int(t)] = d
            self._ptrs[int(t)] = d.data_ptr()

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
    converted on the device). Host arrays should be pinned (see `pinned`) and must stay alive
    until sync() — the pipeline keeps references until then."""

    def __init__(self, rd: RenderData, procs: ProcessorSet, batch: int, length: int, dtype=np.float32, depth: int = 2):
        from . import _tables  # noqa: F401
        self.rd, self.procs = rd, procs
        self.batch, self.length = int(batch), int(length)
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise ValueError("RenderPipeline: dtype must be float32 or float64")
        self._h = ctypes.c_void_p()
        _check(_lib.mg_pipeline_create(rd.handle, procs.handle, self.batch, self.length,
                                       int(self.dtype == np.float32), int(depth), ctypes.byref(self._h)))
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
