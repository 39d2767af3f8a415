"""One mini-batch EM step (forward + backward + EM) on device buffers,
optionally replayed as a CUDA graph.

This is ``train._accumulate_batch`` + ``em_step_full`` + ``em_step_mini`` +
``apply_theta`` of the reference (``pcirc/train.py:84-101, 133-142``) for a
fixed batch size, with every launch issued by the C ABI on the caller's
stream.  With ``graph=True`` the whole step is captured once and replayed:
the batch is copied into a static input buffer, and the per-step log-
likelihood lands in a static device scalar.  The C launch sequence is
graph-safe (no host synchronisation, tensor maps passed as kernel
parameters, caller-owned buffers), so replay and eager launches run the
same kernels on the same data.
"""
from __future__ import annotations

from . import _lib
from .buffers import allocate_buffers
from .em import em_update_
from .plan import device_plan


class TrainStep:
    """Fixed-batch training step.  ``run(x)`` takes an int32 device (or pinned
    host) tensor [B, num_vars] and returns the step's summed log-likelihood
    as a float64 device scalar (the static one when graphed)."""

    def __init__(self, compiled, batch_size: int, *, pseudocount: float, step_size: float,
                 device=None, graph: bool = True, allreduce=None):
        import torch
        self.c = compiled
        self.B = int(batch_size)
        self.pseudocount = float(pseudocount)
        self.step_size = float(step_size)
        self.plan = device_plan(compiled, device)
        self.dev = self.plan.device
        self.bufs = allocate_buffers(compiled, self.B, self.dev, plan=self.plan)
        self.x = torch.zeros((self.B, compiled.num_vars), dtype=torch.int32, device=self.dev)
        self.allreduce = allreduce
        # the step never reads prod_flows: skip writing it when the layout allows
        self._pf_ptr = (0 if self.plan.info.get("prod_flows_optional")
                        else self.bufs.prod_flows_full.data_ptr())
        # one process: no flow all-reduce between backward and EM, so the
        # input-flow pass may apply EM to the inputs' pmfs (pcb_plan_set_inline_em)
        self._inline_em = allreduce is None
        self.lean_mode = 1  # 2: no side-stream overlap (per-kernel profiling)
        self.graph = None
        self.ll = None
        self.launches_per_step = None
        if graph:
            self._capture()

    def _eager(self, x):
        p, b = self.plan, self.bufs
        s = _lib.stream_handle()  # the capture stream while a graph records
        _lib.call("pcb_transpose_batch_i32", p.handle, s, self.B, b.ldb, x.data_ptr(),
                  b.xT.data_ptr())
        # lean launches: the step never reads node values / flows, so aliased
        # leaf products skip their evaluation and push (pcb_plan_set_lean)
        _lib.call("pcb_plan_set_lean", p.handle, self.lean_mode)
        if self._inline_em:
            _lib.call("pcb_plan_set_inline_em", p.handle, 1, self.pseudocount, self.step_size,
                      p.status.data_ptr())
        try:
            _lib.call("pcb_forward", p.handle, s, self.B, b.ldb, b.xT.data_ptr(),
                      p.theta.data_ptr(), b.values_full.data_ptr(), b.scratch_full.data_ptr(),
                      b.lroot.data_ptr(), b.work.data_ptr())
            _lib.call("pcb_backward", p.handle, s, self.B, b.ldb, b.xT.data_ptr(),
                      p.theta.data_ptr(), b.values_full.data_ptr(), b.flows_full.data_ptr(),
                      b.scratch_full.data_ptr(), b.flow_scratch_full.data_ptr(),
                      self._pf_ptr, b.f_params.data_ptr(), b.work.data_ptr())
            ll = b.lroot.double().sum()
            if self.allreduce is not None:
                self.allreduce(b.f_params, ll)
            em_update_(self.c, b.f_params, pseudocount=self.pseudocount,
                       step_size=self.step_size, check=False, plan=p)
        finally:
            _lib.call("pcb_plan_set_lean", p.handle, 0)
            if self._inline_em:
                _lib.call("pcb_plan_set_inline_em", p.handle, 0, 0.0, 1.0, 0)
        return ll

    def _capture(self):
        import torch
        # one eager step on the capture stream builds every lazy kernel attribute
        # (it also advances theta once: restore it afterwards)
        saved = self.plan.theta.clone()
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
        self.graph = g

    def run(self, x):
        if self.graph is None:
            return self._eager(x)
        if x is not self.x:
            self.x.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.ll
