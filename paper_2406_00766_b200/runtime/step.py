"""One mini-batch EM step (forward + backward + EM) on device buffers,
optionally replayed as a CUDA graph.

This is ``train._accumulate_batch`` + ``em_step_full`` + ``em_step_mini`` +
``apply_theta`` of the reference (``pcirc/train.py:84-101, 133-142``) for a
fixed batch size: one ``pcb_train_step`` call on the caller's stream with
lean launches (nothing downstream reads node values / flows) and, in one
process, the EM update applied inside the backward pass where the plan
proves it exact.  With ``graph=True`` the step is captured once and
replayed: the batch is copied into a static input buffer and the per-step
log-likelihood lands in a static device scalar.  The launch sequence is
graph-safe (no host synchronisation, tensor maps passed as kernel
parameters, caller-owned buffers, per-step state in the call's arguments
and this step's ``pcb_exec``), so replay and eager launches run the same
kernels on the same data.

Data parallel (``allreduce`` given): the step runs forward + lean backward
only, the caller's all-reduce sums ``f_params[:theta_size]`` and the
log-likelihood, then ``pcb_em_update`` applies the (replicated) EM kernel.
Full-batch EM (``accumulate`` given): forward + lean backward, the step's
parameter flows added into the epoch accumulator (no EM).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from .buffers import allocate_buffers
from .em import em_update_
from .plan import device_plan


class TrainStep:
    """Fixed-batch training step.  ``run(x)`` takes an int32 device (or pinned
    host) tensor [B, num_vars] and returns the step's summed log-likelihood
    as a float64 device scalar (the static one when graphed)."""

    def __init__(self, compiled, batch_size: int, *, pseudocount: float, step_size: float,
                 device=None, graph: bool = True, allreduce=None, tensor_cores: bool = True,
                 accumulate=None):
        import torch
        self.c = compiled
        self.B = int(batch_size)
        self.pseudocount = float(pseudocount)
        self.step_size = float(step_size)
        self.plan = device_plan(compiled, device, tensor_cores=tensor_cores)
        self.dev = self.plan.device
        self.bufs = allocate_buffers(compiled, self.B, self.dev, plan=self.plan)
        self.x = torch.zeros((self.B, compiled.num_vars), dtype=torch.int32, device=self.dev)
        self.allreduce = allreduce
        self.accumulate = accumulate
        # the step never reads prod_flows: skip writing it when the layout allows
        self._pf_ptr = (0 if self.plan.info.get("prod_flows_optional")
                        else self.bufs.prod_flows_full.data_ptr())
        h = C.c_void_p()
        with torch.cuda.device(self.dev):
            _lib.call("pcb_exec_create", self.plan.handle, C.byref(h))
        self._exec = h
        self.serial = False  # True: no side-stream overlap (per-kernel-class profiling)
        self.graph = None
        self.ll = None
        self.launches_per_step = None
        if graph:
            self._capture()

    def __del__(self):
        h = getattr(self, "_exec", None)
        if h is not None and h.value:
            try:
                _lib.load().pcb_exec_destroy(h)
            except Exception:
                pass

    def _flags(self, em: bool) -> int:
        f = _lib.STEP_LEAN | (_lib.STEP_SERIAL if self.serial else 0)
        return f | (_lib.STEP_EM if em else 0)

    def _eager(self, x):
        p, b = self.plan, self.bufs
        s = _lib.stream_handle()  # the capture stream while a graph records
        _lib.call("pcb_transpose_batch_i32", p.handle, s, self.B, b.ldb, x.data_ptr(),
                  b.xT.data_ptr())
        # one process, mini-batch EM: the EM update inside the step
        one = self.allreduce is None and self.accumulate is None
        _lib.call("pcb_train_step", p.handle, self._exec, s, self.B, b.ldb, b.xT.data_ptr(),
                  p.theta.data_ptr(), b.values_full.data_ptr(), b.flows_full.data_ptr(),
                  b.scratch_full.data_ptr(), b.flow_scratch_full.data_ptr(), self._pf_ptr,
                  b.f_params.data_ptr(), b.lroot.data_ptr(), b.work.data_ptr(),
                  self._flags(one), self.pseudocount, self.step_size, p.status.data_ptr())
        ll = b.lroot.double().sum()
        if self.accumulate is not None:
            _lib.call("pcb_axpy_accumulate", s, self.c.theta_size, b.f_params.data_ptr(),
                      self.accumulate.data_ptr())
        elif not one:
            self.allreduce(b.f_params, ll)
            em_update_(self.c, b.f_params, pseudocount=self.pseudocount,
                       step_size=self.step_size, check=False, plan=p)
        return ll

    def _capture(self):
        import torch
        # one eager step on the capture stream builds every lazy kernel attribute
        # (it also advances theta once: restore it afterwards)
        saved = self.plan.theta.clone()
        saved_acc = self.accumulate.clone() if self.accumulate is not None else None
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self._eager(self.x)
            torch.cuda.synchronize(self.dev)
            g = torch.cuda.CUDAGraph()
            n0 = _lib.load().pcb_launch_count()
            with torch.cuda.graph(g, stream=side):
                self.ll = self._eager(self.x)
            self.launches_per_step = int(_lib.load().pcb_launch_count() - n0)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize(self.dev)
        self.plan.theta.copy_(saved)
        self.plan.refresh_mma()
        if saved_acc is not None:
            self.accumulate.copy_(saved_acc)
        self.graph = g

    def run(self, x):
        self.c.mark_theta_on_device(self.plan)
        if self.graph is None:
            return self._eager(x)
        if x is not self.x:
            self.x.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.ll
