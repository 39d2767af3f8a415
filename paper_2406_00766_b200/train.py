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


def _device_data(compiled, data, dev):
    """A device-resident dataset as int32, validated there (``engine.py:36-52``)."""
    import torch
    from .errors import FormatError
    x = data
    if x.dim() != 2 or x.shape[1] != compiled.num_vars:
        raise FormatError(f"batch must have shape (n, {compiled.num_vars}), got "
                          f"{tuple(x.shape)}")
    x = x.to(dev)
    if x.numel():
        cats = torch.as_tensor(np.asarray(compiled.var_categories), device=dev)
        if bool((x < -1).any()):
            raise FormatError("category values must be >= 0, or -1 for missing")
        bad = (x >= cats[None, :]).any(dim=0)
        if bool(bad.any()):
            var = int(torch.nonzero(bad)[0, 0])
            raise FormatError(
                f"variable {var} has values outside [0, {compiled.var_categories[var]})")
    return x.to(torch.int32).contiguous()


def cached_step(compiled, B: int, *, pseudocount: float, step_size: float, device=None,
                graph: bool = True, tensor_cores: bool = True, group=None, full: bool = False):
    """The training step of batch size B for these settings, built once per
    device plan and reused by every later ``train()`` call (its buffers and
    CUDA graph included).  Data parallel when torch.distributed is
    initialised; ``full``: flows accumulated for full-batch EM."""
    import torch
    from .runtime.plan import device_plan
    from .runtime.step import TrainStep
    plan = device_plan(compiled, device, tensor_cores=tensor_cores)
    cache = plan.__dict__.setdefault("_train_steps", {})
    world = _dp()[1]
    graph = graph and B > 0
    key = (B, float(pseudocount), float(step_size), full, graph, world > 1, id(group))
    ts = cache.get(key)
    if ts is not None:
        return ts
    ar = None
    if world > 1:
        import torch.distributed as dist

        def ar(t):  # in-place sum over the data-parallel group
            dist.all_reduce(t, group=group)
    acc = None
    if full:
        acc_key = ("acc", world > 1, id(group))
        acc = cache.get(acc_key)
        if acc is None:
            acc = cache[acc_key] = torch.zeros(max(compiled.theta_size, 1),
                                               dtype=torch.float32, device=plan.device)
    ts = cache[key] = TrainStep(compiled, B, pseudocount=pseudocount, step_size=step_size,
                                device=plan.device, graph=graph, tensor_cores=tensor_cores,
                                allreduce=None if full else ar, accumulate=acc)
    return ts


def train(compiled, data, cfg: TrainConfig | None = None, *, device=None,
          tensor_cores: bool = True, group=None, graph: bool = True) -> TrainResult:
    """Run EM; ``compiled.theta`` holds the trained table on return (``train.py:104-154``).

    Every step is one ``pcb_train_step`` (``runtime.step.TrainStep``): lean
    launches, EM inside the backward pass where exact (one process), each
    batch size's step captured once as a CUDA graph and replayed (steps are
    cached on the device plan, so later calls reuse them).  Host data stream
    to the device behind the compute (``runtime.loader.HostBatches``: rows
    gathered in epoch order, validated per batch); device data are gathered
    in place.  The epoch log-likelihood and the EM status counters
    accumulate on the device; the host synchronises once per epoch.  If an
    epoch reports a dead EM step or non-finite parameters, it is re-run from
    its starting table eagerly with a check after every step, so the
    ``NumericError`` is raised at the failing step with the parameters of the
    step before it, as the reference does (``em.py:70-75``).
    """
    import torch
    from .errors import FormatError
    from .runtime.em import em_update_, propagate_theta
    from .runtime.loader import DeviceBatches, HostBatches
    from .runtime.plan import device_plan
    cfg = cfg or TrainConfig()
    plan = device_plan(compiled, device, tensor_cores=tensor_cores)
    dev = plan.device
    on_device = isinstance(data, torch.Tensor)
    if not on_device:
        data = np.asarray(data)
        if data.dtype.kind not in "iu":
            data = data.astype(np.int64)
    n = int(data.shape[0]) if data.ndim == 2 else 0
    if n == 0:
        raise UsageError("training data is empty")
    if data.shape[1] != compiled.num_vars:
        raise FormatError(f"batch must have shape (n, {compiled.num_vars}), got "
                          f"{tuple(data.shape)}")
    result = TrainResult()
    batch_size = cfg.batch_size
    if batch_size > n:
        result.notes.append(f"batch size {batch_size} exceeds {n} samples; clipped to {n}")
        batch_size = n
    if not plan.theta_finite:
        raise NumericError("parameter table contains non-finite values")
    rank, world = _dp()
    shuffle_rng = np.random.default_rng(np.random.SeedSequence(cfg.seed).spawn(2)[1])
    theta_size = compiled.theta_size
    n_groups = int(compiled.group_off.size - 1)
    full = cfg.mode == "full"
    # NCCL collectives can be captured in the step's graph; other backends replay eagerly
    use_graph = graph
    if world > 1:
        import torch.distributed as dist
        use_graph = graph and dist.get_backend(group) == "nccl"
    # this rank's row span of every batch (the reference's _chunk_ranges split)
    spans = []
    for a in range(0, n, batch_size):
        lo, hi = shard_span(min(n, a + batch_size) - a, rank, world)
        spans.append((a + lo, a + hi))
    with torch.cuda.device(dev):
        data_dev = _device_data(compiled, data, dev) if on_device else None

        def step_for(B, graphed):
            return cached_step(compiled, B, pseudocount=cfg.pseudocount,
                               step_size=cfg.step_size, device=dev, graph=graphed,
                               tensor_cores=tensor_cores, group=group, full=full)

        def acc():  # the full-batch accumulator shared by the cached steps
            return step_for(spans[0][1] - spans[0][0], use_graph).accumulate

        def run_epoch(order, graphed: bool, prev=None):
            """prev: eager re-run with a check after every step (the table
            before each step is kept in prev)."""
            if on_device:
                src = DeviceBatches(data_dev, torch.from_numpy(order).to(dev), spans)
            else:
                src = HostBatches(data, order, spans, compiled.var_categories, dev)
            ep_ll = torch.zeros((), dtype=torch.float64, device=dev)
            dead = torch.zeros((), dtype=torch.int32, device=dev)
            bad = torch.zeros((), dtype=torch.int32, device=dev)
            if full:
                acc().zero_()
            try:
                for i, (a, b) in enumerate(spans):
                    ts = step_for(b - a, graphed)
                    src.fill(i, ts.x)
                    if prev is not None and not full:
                        prev.copy_(plan.theta)
                    ep_ll += ts.run(ts.x)
                    if full:
                        continue
                    if n_groups:
                        dead += (plan.status[0] == 0).int()
                    bad += plan.status[1]
                    if prev is not None and (int(dead.item()) or int(bad.item())):
                        return ep_ll, dead, bad, True
            finally:
                src.close()
            if full:
                allreduce_accumulators(acc(), ep_ll, theta_size, group)
                em_update_(compiled, acc(), pseudocount=cfg.pseudocount, step_size=1.0,
                           check=False, plan=plan)
                if n_groups:
                    dead += (plan.status[0] == 0).int()
                bad += plan.status[1]
            return ep_ll, dead, bad, False

        snapshot = None
        for _ in range(cfg.epochs):
            t0 = time.perf_counter()
            order = shuffle_rng.permutation(n) if cfg.mode == "mini" else np.arange(n)
            if snapshot is None:
                snapshot = plan.theta.clone()
            else:
                snapshot.copy_(plan.theta)
            try:
                ep_ll, dead, bad, _ = run_epoch(order, use_graph)
            except FormatError:
                propagate_theta(compiled, plan)
                raise
            if int(dead.item()) or int(bad.item()):
                # re-run the epoch from its starting table with per-step
                # checks: raise at the failing step, parameters of the step
                # before it (the failing step's update is rolled back)
                plan.theta.copy_(snapshot)
                plan.refresh_mma()
                prev = torch.empty_like(plan.theta)
                ep_ll, dead, bad, stopped = run_epoch(order, False, prev=prev)
                if stopped and not full:
                    plan.theta.copy_(prev)
                    plan.refresh_mma()
                plan.theta_finite = bool(torch.isfinite(plan.theta).all().item())
                propagate_theta(compiled, plan)
                if int(dead.item()):
                    raise NumericError("every normalization group accumulated zero flow; "
                                       "use a positive pseudocount or check the data")
                raise NumericError("EM update produced non-finite parameters")
            ll = float(ep_ll.item())
            result.epoch_log_likelihood.append(ll / n)
            result.epoch_seconds.append(time.perf_counter() - t0)
        propagate_theta(compiled, plan)
    return result
