"""EM training on the device (drop-in for ``pcirc/train.py``).

The dataset is validated once and made resident on the GPU as int32; each
step gathers its rows, runs ``pcb_forward`` + ``pcb_backward`` and, in
mini-batch mode, one fused renormalise-and-blend EM kernel
(``pcb_em_update``).  Nothing returns to the host inside an epoch: the
epoch log-likelihood accumulates on the device and EM failures (a step in
which no group carried flow) are counted on the device and raised as
``NumericError`` at the end of the epoch.

Data parallel (one process per GPU, ``torch.distributed`` initialised by
the caller, e.g. under torchrun): every rank holds the full circuit, takes
the contiguous span ``shard_span(B, rank, world)`` of each batch (the
reference's ``_chunk_ranges`` split, ``train.py:78-81``), and the only
collective is one all-reduce of ``f_params[:theta_size]`` plus the batch
log-likelihood before the (replicated, deterministic) EM kernel — the
reference's fixed-order worker merge (``train.py:100-101``) becomes an NCCL
sum.  Full-batch mode all-reduces once per epoch.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import NumericError, UsageError

__all__ = ["TrainConfig", "TrainResult", "default_threads", "train", "shard_span",
           "allreduce_accumulators"]


def default_threads() -> int:
    return os.cpu_count() or 1


@dataclass
class TrainConfig:
    """Same fields and validation as ``train.py:38-60``; ``threads`` is
    accepted for compatibility (GPU work is not split across host threads)."""

    epochs: int = 1
    batch_size: int = 256
    mode: str = "full"
    step_size: float = 0.01
    pseudocount: float = 0.0
    seed: int = 0
    threads: int | None = None

    def __post_init__(self):
        if self.epochs < 1:
            raise UsageError(f"epochs must be >= 1, got {self.epochs}")
        if self.batch_size < 1:
            raise UsageError(f"batch size must be >= 1, got {self.batch_size}")
        if self.mode not in {"full", "mini"}:
            raise UsageError(f"em mode must be 'full' or 'mini', got {self.mode!r}")
        if not 0.0 < self.step_size <= 1.0:
            raise UsageError(f"step size must be in (0, 1], got {self.step_size}")
        if self.pseudocount < 0:
            raise UsageError(f"pseudocount must be >= 0, got {self.pseudocount}")
        if self.threads is not None and self.threads < 1:
            raise UsageError(f"threads must be >= 1, got {self.threads}")


@dataclass
class TrainResult:
    epoch_log_likelihood: list = field(default_factory=list)
    epoch_seconds: list = field(default_factory=list)
    notes: list = field(default_factory=list)

    def log_lines(self) -> list:
        return [f"epoch={i + 1} ll={ll:.10f} seconds={s:.3f}"
                for i, (ll, s) in enumerate(zip(self.epoch_log_likelihood, self.epoch_seconds))]


def shard_span(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous span of ``n`` samples owned by ``rank`` (``train.py:78-81``)."""
    parts = max(1, min(world, n))
    bounds = np.linspace(0, n, parts + 1).astype(int)
    if rank >= parts:
        return int(n), int(n)
    return int(bounds[rank]), int(bounds[rank + 1])


def allreduce_accumulators(f_params, ll, theta_size: int, group=None):
    """Sum the parameter flows (theta prefix only; replica ranges are already
    reduced locally) and the log-likelihood over the data-parallel group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(f_params[:theta_size], group=group)
        dist.all_reduce(ll, group=group)


def _dp():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def train(compiled, data, cfg: TrainConfig | None = None, *, device=None,
          tensor_cores: bool = True, group=None) -> TrainResult:
    """Run EM; ``compiled.theta`` holds the trained table on return (``train.py:104-154``)."""
    import torch
    from .runtime import _lib
    from .runtime.buffers import allocate_buffers
    from .runtime.em import em_update_, sync_theta_to_host
    from .runtime.engine import _validate_host_batch
    from .runtime.plan import device_plan

    cfg = cfg or TrainConfig()
    data = np.asarray(data, dtype=np.int64)
    n = data.shape[0] if data.ndim == 2 else 0
    if n == 0:
        raise UsageError("training data is empty")
    data = _validate_host_batch(compiled, data)
    result = TrainResult()
    batch_size = cfg.batch_size
    if batch_size > n:
        result.notes.append(f"batch size {batch_size} exceeds {n} samples; clipped to {n}")
        batch_size = n
    plan = device_plan(compiled, device, tensor_cores=tensor_cores)
    if not plan.theta_finite:
        raise NumericError("parameter table contains non-finite values")
    rank, world = _dp()
    dev = plan.device
    data_dev = torch.from_numpy(data.astype(np.int32)).to(dev)
    shuffle_rng = np.random.default_rng(np.random.SeedSequence(cfg.seed).spawn(2)[1])
    theta_size = compiled.theta_size
    n_groups = int(compiled.group_off.size - 1)
    bufs_cache: dict = {}
    with torch.cuda.device(dev):
        stream = _lib.stream_handle()
        dead_steps = torch.zeros((), dtype=torch.int32, device=dev)
        bad_values = torch.zeros((), dtype=torch.int32, device=dev)
        for _ in range(cfg.epochs):
            t0 = time.perf_counter()
            order = shuffle_rng.permutation(n) if cfg.mode == "mini" else np.arange(n)
            order_dev = torch.from_numpy(order).to(dev)
            ep_ll = torch.zeros((), dtype=torch.float64, device=dev)
            ep_fp = (torch.zeros(compiled.f_params_size, dtype=torch.float32, device=dev)
                     if cfg.mode == "full" else None)
            samples = 0
            for a in range(0, n, batch_size):
                b_all = min(n, a + batch_size) - a
                lo, hi = shard_span(b_all, rank, world)
                B = hi - lo
                bufs = bufs_cache.get(B)
                if bufs is None:
                    bufs = bufs_cache[B] = allocate_buffers(compiled, B, dev, plan=plan)
                idx = order_dev[a + lo:a + hi]
                xb = data_dev.index_select(0, idx)
                step_ll = torch.zeros((), dtype=torch.float64, device=dev)
                if B:
                    _lib.call("pcb_transpose_batch_i32", plan.handle, stream, B, bufs.ldb,
                              xb.data_ptr(), bufs.xT.data_ptr())
                    _lib.call("pcb_forward", plan.handle, stream, B, bufs.ldb,
                              bufs.xT.data_ptr(), plan.theta.data_ptr(),
                              bufs.values_full.data_ptr(), bufs.scratch_full.data_ptr(),
                              bufs.lroot.data_ptr(), bufs.work.data_ptr())
                    step_ll += bufs.lroot.double().sum()
                _lib.call("pcb_backward", plan.handle, stream, B, bufs.ldb, bufs.xT.data_ptr(),
                          plan.theta.data_ptr(), bufs.values_full.data_ptr(),
                          bufs.flows_full.data_ptr(), bufs.scratch_full.data_ptr(),
                          bufs.flow_scratch_full.data_ptr(), bufs.prod_flows_full.data_ptr(),
                          bufs.f_params.data_ptr(), bufs.work.data_ptr())
                samples += b_all
                if cfg.mode == "full":
                    _lib.call("pcb_axpy_accumulate", stream, ep_fp.numel(),
                              bufs.f_params.data_ptr(), ep_fp.data_ptr())
                    ep_ll += step_ll
                    continue
                allreduce_accumulators(bufs.f_params, step_ll, theta_size, group)
                ep_ll += step_ll
                em_update_(compiled, bufs.f_params, pseudocount=cfg.pseudocount,
                           step_size=cfg.step_size, check=False, plan=plan)
                if n_groups:
                    dead_steps += (plan.status[0] == 0).int()
                bad_values += plan.status[1]
            if cfg.mode == "full":
                allreduce_accumulators(ep_fp, ep_ll, theta_size, group)
                em_update_(compiled, ep_fp, pseudocount=cfg.pseudocount, step_size=1.0,
                           check=False, plan=plan)
                if n_groups:
                    dead_steps += (plan.status[0] == 0).int()
                bad_values += plan.status[1]
            ll = float(ep_ll.item())
            if int(dead_steps.item()):
                raise NumericError("every normalization group accumulated zero flow; "
                                   "use a positive pseudocount or check the data")
            if int(bad_values.item()):
                raise NumericError("EM update produced non-finite parameters")
            result.epoch_log_likelihood.append(ll / samples)
            result.epoch_seconds.append(time.perf_counter() - t0)
        sync_theta_to_host(compiled, dev)
    return result
