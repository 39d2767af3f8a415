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

Data parallel (``allreduce`` given: a callable summing a device tensor in
place over the ranks, e.g. an NCCL ``all_reduce``): the step runs forward +
lean backward only, ``f_params[:theta_size]`` and the log-likelihood are
summed, then ``pcb_em_update`` applies the (replicated) EM kernel.  The sum
is bucketed by layer: the backward pass records an event as each sum
layer's parameter flows are issued (``pcb_exec_set_flow_events``), and the
all-reduce of that layer's f_params range starts on a communication stream
at that event, overlapping the lower layers' backward; the input pmfs and
the zero tile follow the input flows.  (Bucketing needs the plan's disjoint
per-layer flow ranges, ``fp_cover``; otherwise one all-reduce at the end.)
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
        # the step never reads prod_flows: skip it when the layout allows
        optional = bool(self.plan.info.get("prod_flows_optional"))
        self.bufs = allocate_buffers(compiled, self.B, self.dev, plan=self.plan,
                                     prod_flows=not optional)
        self.x = torch.zeros((self.B, compiled.num_vars), dtype=torch.int32, device=self.dev)
        self.allreduce = allreduce
        self.accumulate = accumulate
        self._pf_ptr = 0 if optional else self.bufs.prod_flows_full.data_ptr()
        h = C.c_void_p()
        with torch.cuda.device(self.dev):
            _lib.call("pcb_exec_create", self.plan.handle, C.byref(h))
            self._exec = h
            self._buckets = None
            if allreduce is not None and accumulate is None:
                self._setup_buckets()
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

    def _setup_buckets(self):
        """Per-layer f_params ranges reduced as each layer finishes, then the
        rest of [0, theta_size) (input pmfs, zero tile) after the input flows."""
        import torch
        info = self.plan.info
        nl = len(self.c.layers)
        theta = self.c.theta_size
        ranges = info["layer_flow_ranges"] if info.get("fp_cover") else [(0, 0)] * nl
        covered = sorted((lo, hi) for lo, hi in ranges if hi > lo)
        rest, pos = [], 0
        for lo, hi in covered:
            if lo > pos:
                rest.append((pos, lo))
            pos = max(pos, hi)
        if pos < theta:
            rest.append((pos, theta))
        self._events = [torch.cuda.Event() for _ in range(nl + 1)]
        for e in self._events:  # materialise the CUDA events
            e.record()
        handles = (C.c_void_p * (nl + 1))(*[e.cuda_event for e in self._events])
        _lib.call("pcb_exec_set_flow_events", self._exec, handles, nl + 1)
        self._buckets = ([(li, lo, hi) for li, (lo, hi) in enumerate(ranges) if hi > lo][::-1]
                         + [(nl, lo, hi) for lo, hi in rest])
        self._comm = torch.cuda.Stream(self.dev)

    def _reduce(self, ll):
        """Bucketed all-reduce of f_params[:theta_size] and the step LL."""
        import torch
        b = self.bufs
        comp = torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(self._comm):
            for li, lo, hi in self._buckets:
                self._comm.wait_event(self._events[li])
                self.allreduce(b.f_params[lo:hi])
            self._comm.wait_stream(comp)  # the LL sum is formed on the compute stream
            self.allreduce(ll)
        comp.wait_stream(self._comm)

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
            self._reduce(ll)
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

    def validate(self, x) -> None:
        """Shape / dtype / device checks and the category check of
        ``engine.py:36-52`` on the device (``pcb_check_batch``): FormatError.
        ``run`` does not validate (the graph replays without host syncs;
        ``train()`` validates every batch before its step)."""
        import torch
        from ..errors import FormatError
        if not isinstance(x, torch.Tensor) or x.shape != (self.B, self.c.num_vars) or \
                x.dtype != torch.int32:
            raise FormatError(f"a step batch is an int32 tensor of shape ({self.B}, "
                              f"{self.c.num_vars})")
        xd = x.to(self.dev)
        b = self.bufs
        s = _lib.stream_handle()
        _lib.call("pcb_transpose_batch_i32", self.plan.handle, s, self.B, b.ldb, xd.data_ptr(),
                  b.xT.data_ptr())
        bad = self.plan.status[3:4]
        bad.zero_()
        _lib.call("pcb_check_batch", self.plan.handle, s, self.B, b.ldb, b.xT.data_ptr(),
                  bad.data_ptr())
        if int(bad.item()):
            raise FormatError("category values must lie in [0, ncat) or be -1 for missing")

    def run(self, x, *, validate: bool = False):
        """One step on batch ``x``; ``validate=True`` checks it first (a
        host synchronisation)."""
        if validate:
            self.validate(x)
        self.c.mark_theta_on_device(self.plan)
        if self.graph is None:
            return self._eager(x)
        if x is not self.x:
            self.x.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.ll
