"""forward / backward on sm_100a (drop-in for ``pcirc/runtime/engine.py``).

``forward(compiled, batch)`` validates the batch like ``engine.py:36-52``,
stages it on the device as a transposed int32 [vars x ldb] table and runs
the whole layered program in one C-ABI call (``pcb_forward``): input
gathers, product gather-adds, tcgen05 sum-layer contractions.  ``backward``
runs ``pcb_backward``: recomputed products, parameter flows, child flows,
flow pushes, input flows and the replica reduction.  Results stay on the
device; ``EvalBuffers`` exposes them as torch tensors.
"""
from __future__ import annotations

import numpy as np

from ..errors import FormatError, NumericError, UsageError
from . import _lib
from .buffers import EvalBuffers, allocate_buffers
from .plan import device_plan

__all__ = ["MISSING", "forward", "backward", "stage_batch"]

MISSING = -1


def _validate_host_batch(compiled, batch) -> np.ndarray:
    """Shape and category checks (``engine.py:36-52``)."""
    data = np.asarray(batch, dtype=np.int64)
    if data.ndim == 1:
        data = data[None, :]
    if data.ndim != 2 or data.shape[1] != compiled.num_vars:
        raise FormatError(f"batch must have shape (n, {compiled.num_vars}), got {data.shape}")
    if data.size and data.min() < MISSING:
        raise FormatError("category values must be >= 0, or -1 for missing")
    cats = np.asarray(compiled.var_categories)[None, :]
    if data.size and np.any(data >= cats):
        var = int(np.argwhere(data >= cats)[0, 1])
        raise FormatError(
            f"variable {var} has values outside [0, {compiled.var_categories[var]})")
    return data


def stage_batch(compiled, plan, batch, bufs: EvalBuffers, *, validate: bool = True):
    """Copy a [B x vars] batch (numpy or torch) into ``bufs.xT`` on the device."""
    import torch
    stream = _lib.stream_handle()
    B, ldb = bufs.batch_size, bufs.ldb
    if isinstance(batch, torch.Tensor) and batch.is_cuda:
        x = batch
        if x.dim() == 1:
            x = x[None, :]
        if x.dim() != 2 or x.shape[1] != compiled.num_vars:
            raise FormatError(
                f"batch must have shape (n, {compiled.num_vars}), got {tuple(x.shape)}")
        x = x.contiguous()
        if x.dtype == torch.int64:
            _lib.call("pcb_transpose_batch_i64", plan.handle, stream, B, ldb, x.data_ptr(),
                      bufs.xT.data_ptr())
        elif x.dtype == torch.int32:
            _lib.call("pcb_transpose_batch_i32", plan.handle, stream, B, ldb, x.data_ptr(),
                      bufs.xT.data_ptr())
        else:
            raise FormatError("device batches must be int32 or int64")
        if validate:
            bad = plan.status[3:4]
            bad.zero_()
            _lib.call("pcb_check_batch", plan.handle, stream, B, ldb, bufs.xT.data_ptr(),
                      bad.data_ptr())
            if int(bad.item()):
                raise FormatError("category values must lie in [0, ncat) or be -1 for missing")
        bufs.batch = None
        return
    data = _validate_host_batch(compiled, batch) if validate else np.asarray(batch)
    xt = np.ascontiguousarray(data.T.astype(np.int32))
    bufs.xT[: xt.shape[0], :B].copy_(torch.from_numpy(xt), non_blocking=False)
    bufs.batch = data


def _batch_rows(compiled, batch) -> int:
    import torch
    if isinstance(batch, torch.Tensor):
        return 1 if batch.dim() == 1 else int(batch.shape[0])
    arr = np.asarray(batch)
    if arr.ndim == 1:
        return 1
    if arr.ndim != 2:
        raise FormatError(f"batch must have shape (n, {compiled.num_vars}), got {arr.shape}")
    return int(arr.shape[0])


def forward(compiled, batch, *, batch_tile: int = 64, bufs: EvalBuffers | None = None,
            device=None, validate: bool = True, tensor_cores: bool = True):
    """Per-sample root log-probabilities; returns ``(lroot, bufs)`` (``engine.py:186-217``).

    ``lroot`` is a float32 CUDA tensor of shape (B,).  ``batch_tile`` is
    accepted for signature compatibility; tiling is fixed by the kernels.
    """
    import torch
    plan = device_plan(compiled, device, tensor_cores=tensor_cores)
    if not plan.theta_finite:
        raise NumericError("parameter table contains non-finite values")
    B = _batch_rows(compiled, batch)
    if bufs is None or bufs.batch_size != B:
        bufs = allocate_buffers(compiled, B, plan.device, plan=plan)
    with torch.cuda.device(plan.device):
        stage_batch(compiled, plan, batch, bufs, validate=validate)
        _lib.call("pcb_forward", plan.handle, _lib.stream_handle(), B, bufs.ldb,
                  bufs.xT.data_ptr(), plan.theta.data_ptr(), bufs.values_full.data_ptr(),
                  bufs.scratch_full.data_ptr(), _lib.ptr(bufs.lroot) if B else 0,
                  bufs.work.data_ptr())
    bufs.forward_done = True
    bufs.backward_done = False
    return bufs.lroot, bufs


def backward(compiled, bufs: EvalBuffers, *, batch_tile: int = 64, device=None,
             tensor_cores: bool = True) -> EvalBuffers:
    """Node and parameter flows of the last forward batch (``engine.py:220-259``)."""
    import torch
    if not bufs.forward_done:
        raise UsageError("backward requires a completed forward pass")
    plan = device_plan(compiled, device if device is not None else bufs.device,
                       tensor_cores=tensor_cores)
    with torch.cuda.device(plan.device):
        _lib.call("pcb_backward", plan.handle, _lib.stream_handle(), bufs.batch_size, bufs.ldb,
                  bufs.xT.data_ptr(), plan.theta.data_ptr(), bufs.values_full.data_ptr(),
                  bufs.flows_full.data_ptr(), bufs.scratch_full.data_ptr(),
                  bufs.flow_scratch_full.data_ptr(), bufs.prod_flows_full.data_ptr(),
                  bufs.f_params.data_ptr(), bufs.work.data_ptr())
    bufs.backward_done = True
    return bufs


def layer_forward(compiled, layer: int, bufs: EvalBuffers, *, tensor_cores: bool = True):
    """Products + sum contraction of one layer (the reference's private
    ``_eval_products`` + ``_forward_group`` pair, ``engine.py:68-102``)."""
    plan = device_plan(compiled, bufs.device, tensor_cores=tensor_cores)
    _lib.call("pcb_layer_forward", plan.handle, layer, _lib.stream_handle(), bufs.batch_size,
              bufs.ldb, plan.theta.data_ptr(), bufs.values_full.data_ptr(),
              bufs.scratch_full.data_ptr(), bufs.work.data_ptr())


def layer_backward(compiled, layer: int, bufs: EvalBuffers, *, tensor_cores: bool = True):
    """Parameter + child flows of one layer (``engine.py:105-165, 249-254``)."""
    plan = device_plan(compiled, bufs.device, tensor_cores=tensor_cores)
    _lib.call("pcb_layer_backward", plan.handle, layer, _lib.stream_handle(), bufs.batch_size,
              bufs.ldb, plan.theta.data_ptr(), bufs.values_full.data_ptr(),
              bufs.flows_full.data_ptr(), bufs.scratch_full.data_ptr(),
              bufs.flow_scratch_full.data_ptr(), bufs.prod_flows_full.data_ptr(),
              bufs.f_params.data_ptr(), bufs.work.data_ptr())
