"""EM updates on the device (drop-in for ``pcirc/runtime/em.py``).

``em_step_full`` renormalises every simplex group of the accumulated flows
(``em.py:58-81``) with the segmented warp-per-group kernel
(``pcb_em_update`` with step 1 on a copy of theta); ``em_step_mini`` blends
(``em.py:84-88``); ``apply_theta`` installs a table (``em.py:91-94``).  The
training loop uses :func:`em_update_` instead, which renormalises and blends
in place in one kernel pass.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..errors import NumericError, UsageError
from . import _lib
from .plan import device_plan

__all__ = ["EMAccumulator", "apply_theta", "em_accumulate", "em_step_full", "em_step_mini",
           "em_update_", "propagate_theta", "sync_theta_to_host", "write_back_params"]


@dataclass
class EMAccumulator:
    """Running sum of parameter flows across batches (``em.py:28-45``)."""

    f_params: object
    batches: int = 0
    samples: int = 0
    _ll: object = None

    @classmethod
    def for_circuit(cls, compiled, device=None) -> "EMAccumulator":
        import torch
        plan = device_plan(compiled, device)
        return cls(f_params=torch.zeros(compiled.f_params_size, dtype=torch.float32,
                                        device=plan.device),
                   _ll=torch.zeros((), dtype=torch.float64, device=plan.device))

    @property
    def log_likelihood(self) -> float:
        return float(self._ll.item()) if self._ll is not None else 0.0

    @log_likelihood.setter
    def log_likelihood(self, v: float) -> None:
        self._ll.fill_(float(v))

    def reset(self):
        self.f_params.zero_()
        self.batches = 0
        self.samples = 0
        self._ll.zero_()


def em_accumulate(acc: EMAccumulator, bufs) -> EMAccumulator:
    if not bufs.backward_done:
        raise UsageError("accumulate requires a completed backward pass")
    _lib.call("pcb_axpy_accumulate", _lib.stream_handle(), acc.f_params.numel(),
              bufs.f_params.data_ptr(), acc.f_params.data_ptr())
    acc.batches += 1
    acc.samples += bufs.batch_size
    if bufs.batch_size:
        acc._ll += bufs.lroot.double().sum()
    return acc


def _status_check(plan, n_groups: int) -> None:
    st = plan.status[:2].cpu()
    if n_groups > 0 and int(st[0]) == 0:
        raise NumericError("every normalization group accumulated zero flow; "
                           "use a positive pseudocount or check the data")
    if int(st[1]):
        raise NumericError("EM update produced non-finite parameters")


def em_update_(compiled, f_params, *, pseudocount: float, step_size: float, theta=None,
               check: bool = True, device=None, plan=None):
    """In-place ``theta <- (1-a) theta + a normalise(F + k)`` over every group
    (on ``plan.theta`` unless another table is given)."""
    if plan is None:
        plan = device_plan(compiled, device if device is not None else f_params.device)
    target = plan.theta if theta is None else theta
    _lib.call("pcb_em_update", plan.handle, _lib.stream_handle(), f_params.data_ptr(),
              target.data_ptr(), float(pseudocount), float(step_size), plan.status.data_ptr())
    if target is plan.theta:
        compiled.mark_theta_on_device(plan)
    # on plan.theta the EM pass rewrites the tensor-core planes itself
    if check:
        _status_check(plan, int(compiled.group_off.size - 1))
    return target


def em_step_full(compiled, acc: EMAccumulator, *, pseudocount: float = 0.0):
    """Renormalised table from accumulated flows; uninformative groups keep theta."""
    if pseudocount < 0:
        raise UsageError(f"pseudocount must be >= 0, got {pseudocount}")
    plan = device_plan(compiled, acc.f_params.device)
    new = plan.theta.clone()
    em_update_(compiled, acc.f_params, pseudocount=pseudocount, step_size=1.0, theta=new,
               plan=plan)
    return new


def em_step_mini(theta, theta_new, step_size: float):
    """``(1 - a) * theta + a * theta_new`` (``em.py:84-88``)."""
    if not 0.0 < step_size <= 1.0:
        raise UsageError(f"step size must be in (0, 1], got {step_size}")
    import torch
    if isinstance(theta, np.ndarray) and isinstance(theta_new, np.ndarray):
        return (1.0 - step_size) * theta + step_size * theta_new
    t = torch.as_tensor(theta, device=getattr(theta_new, "device", None))
    return (1.0 - step_size) * t + step_size * torch.as_tensor(theta_new, device=t.device)


def apply_theta(compiled, new_theta):
    """Install a parameter table on the host copy and every device plan."""
    import torch
    size = compiled.theta_size
    shape = tuple(new_theta.shape)
    if shape != (size,):
        raise UsageError("parameter table shape mismatch")
    if isinstance(new_theta, torch.Tensor):
        host = new_theta.detach().double().cpu().numpy()
    else:
        host = np.asarray(new_theta, dtype=np.float64)
    compiled.theta[:] = host
    for plan in (compiled._device_plans or {}).values():
        plan.upload_theta(new_theta if isinstance(new_theta, torch.Tensor) else compiled.theta)


def sync_theta_to_host(compiled, device=None, *, plan=None) -> np.ndarray:
    """Copy a plan's device theta (authoritative during training) back to
    ``compiled.theta`` now (it is otherwise synced lazily on access)."""
    plan = plan if plan is not None else device_plan(compiled, device)
    compiled.mark_theta_on_device(plan)
    return compiled.theta


def propagate_theta(compiled, plan) -> None:
    """After training ``plan``: every other device plan of ``compiled`` (the
    other tensor-core setting, other devices) takes its table, and the host
    copy follows lazily."""
    for other in (compiled._device_plans or {}).values():
        if other is plan:
            continue
        other.upload_theta(plan.theta)
    compiled.mark_theta_on_device(plan)


def write_back_params(compiled, graph):
    """Trained physical parameters onto the logical graph slots (``em.py:97-100``)."""
    slots = np.flatnonzero(compiled.slot_phys >= 0)
    graph.set_param_values(slots, compiled.theta[compiled.slot_phys[slots]])
