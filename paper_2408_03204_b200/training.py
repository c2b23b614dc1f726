"""Optimisation config (BASELINE configs 4/5): analytic parameter gradients + plain gradient
descent, one process per GPU, shared parameters all-reduced over NCCL.

The reference optimises with central differences (`fit.cpp:25-96`): two full renders per
trainable scalar per step, MSE loss, plain gradient descent, dynamics rows projected into
their legal ranges (`fit.cpp:13-21`). Here one forward + one reverse-mode pass
(DeviceRenderer.backward, mg_render_backward_arena) gives every gradient at once; the MSE
loss/gradient and the update run as library kernels (mg_mse_loss_grad, mg_sgd_step).

Multi-GPU: every rank holds the same parameter set and renders its own sources (data
parallel over the audio); the per-type gradient tables are views into ONE flat fp64 buffer,
so a step needs exactly one all-reduce (torch.distributed, NCCL over NVLink). It is the
only collective of the whole path (the forward render has none).
"""
from __future__ import annotations

import ctypes
from typing import Dict, Iterable, Optional, Sequence, Tuple

import numpy as np
import torch

from . import (NodeType, ProcessorSet, RenderData, _check, _lib, _u64, _vp, compute_render_data, param_width)
from .device import DeviceRenderer

_lib.mg_mse_scratch_bytes.restype = ctypes.c_uint64
_lib.mg_mse_scratch_bytes.argtypes = []
_lib.mg_mse_loss_grad.restype = ctypes.c_int32
_lib.mg_mse_loss_grad.argtypes = [_vp, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp]
_lib.mg_sgd_step.restype = ctypes.c_int32
_lib.mg_sgd_step.argtypes = [ctypes.c_int32, _vp, _vp, ctypes.c_int32, ctypes.c_double, _vp]


def reduce_gradients(flat: torch.Tensor, group=None) -> int:
    """Sum the flat gradient buffer over the ranks of `group` (one all-reduce; NCCL on GPUs,
    gloo in the CPU tests) and return the world size to average by."""
    if group is None:
        return 1
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return world


class Trainer:
    """One optimisation step = render -> MSE loss + output gradient -> backward -> (all-reduce
    of the flat gradient buffer, averaged over ranks) -> gradient step on the trainable types.
    `params`: render-order tables (RenderData.reorder_params). `group`: a torch.distributed
    process group (NCCL) or None for a single GPU."""

    def __init__(self, rd: RenderData, procs: ProcessorSet, batch: int, length: int, params: Dict[int, np.ndarray],
                 trainable: Iterable[int] = (NodeType.GAIN,), learning_rate: float = 0.5, group=None,
                 device: Optional[torch.device] = None):
        self.rd, self.procs = rd, procs
        self.trainable = [int(t) for t in trainable]
        for t in self.trainable:
            if param_width(t) == 0:
                raise ValueError(f"fit: '{NodeType(t).name.lower()}' has no parameters")
        self.lr = float(learning_rate)
        self.group = group
        self.dr = DeviceRenderer(rd, procs, batch, length, params, device=device, backward=True)
        dev = self.dr.device
        sizes = {t: tab.numel() for t, tab in self.dr.tables.items()}
        self.flat = torch.zeros(max(1, sum(sizes.values())), dtype=torch.float64, device=dev)
        self.grads: Dict[int, torch.Tensor] = {}
        off = 0
        for t, tab in self.dr.tables.items():
            self.grads[t] = self.flat[off:off + sizes[t]].view(tab.shape)
            off += sizes[t]
        n_out = rd.buffer_rows - rd.output_begin
        self.grad_out = torch.empty((n_out, batch, 2, length), dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.scratch = torch.empty(int(_lib.mg_mse_scratch_bytes()), dtype=torch.uint8, device=dev)
        self.world = 1
        if group is not None:
            import torch.distributed as dist
            self.world = dist.get_world_size(group)

    @property
    def params(self) -> Dict[int, torch.Tensor]:
        return self.dr.tables

    def step(self, sources: torch.Tensor, target: torch.Tensor, update: bool = True) -> torch.Tensor:
        """Enqueue one step on the current stream; returns the device loss (before the update)."""
        s = torch.cuda.current_stream(self.dr.device)
        self.dr.sources.copy_(sources)
        out = self.dr.render(s)
        _check(_lib.mg_mse_loss_grad(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(target.data_ptr()), out.numel(),
                                     ctypes.c_void_p(self.grad_out.data_ptr()), ctypes.c_void_p(self.loss.data_ptr()),
                                     ctypes.c_void_p(self.scratch.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
        self.dr.backward(self.grad_out, s, grads=self.grads)
        lr = self.lr / reduce_gradients(self.flat, self.group)  # mean of the ranks' gradients
        if update:
            for t in self.trainable:
                tab = self.dr.tables.get(t)
                if tab is None:
                    continue
                _check(_lib.mg_sgd_step(t, ctypes.c_void_p(tab.data_ptr()), ctypes.c_void_p(self.grads[t].data_ptr()),
                                        tab.shape[0], lr, ctypes.c_void_p(s.cuda_stream)))
        return self.loss


def fit(fg, init: Dict[int, np.ndarray], procs: ProcessorSet, sources: np.ndarray, target: np.ndarray,
        trainable: Sequence[int] = (NodeType.GAIN,), steps: int = 200, learning_rate: float = 0.5,
        device: Optional[torch.device] = None) -> Tuple[Dict[NodeType, np.ndarray], np.ndarray]:
    """`fit.cpp:25-96` with analytic gradients: MSE between the outputs and `target`
    ([num_outputs][B][2][L]), `steps` plain gradient steps on the trainable types (every type
    with parameters is trainable here; the reference limits itself to the small ones because
    of finite-difference cost), dynamics rows projected after each step. Returns (params in
    original row order, loss history: the loss before each step, then the final loss)."""
    rd = compute_render_data(fg)
    src = np.asarray(sources, dtype=np.float64)
    tgt = np.asarray(target, dtype=np.float64)
    if tgt.shape[0] != rd.buffer_rows - rd.output_begin:
        raise ValueError("fit: target must have one buffer per out node")
    if tgt.shape[1:] != src.shape[1:]:
        raise ValueError("fit: target shape mismatch")
    k, b, _, n = src.shape
    tr = Trainer(rd, procs, b, n, rd.reorder_params(init), trainable, learning_rate, device=device)
    dev = tr.dr.device
    s_dev = torch.as_tensor(src, dtype=torch.float32).to(dev)
    t_dev = torch.as_tensor(tgt, dtype=torch.float32).to(dev)
    hist = []
    for _ in range(steps):
        hist.append(float(tr.step(s_dev, t_dev).item()))
    hist.append(float(tr.step(s_dev, t_dev, update=False).item()))
    params = rd.original_order({t: v.cpu().numpy() for t, v in tr.params.items()})
    return params, np.asarray(hist)
