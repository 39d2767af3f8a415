"""Device batch workspace (drop-in for ``pcirc/runtime/buffers.py:18-57``).

Same arrays, same (rows x batch) node-major layout, on the GPU in fp32.
Rows are padded to a stride ``ldb`` (multiple of 32 samples) so kernels
can vectorise; the public attributes are ``[:, :B]`` views, so
``bufs.values[slot, col]`` indexes exactly like the reference.

The device stores log values as (integer block base, fp32 offset) pairs
(csrc/pcb_internal.cuh): ``values_full`` holds the offsets and the work
buffer the per-(sum block, sample) bases.  ``bufs.values`` adds them back
(fp32 log values, as the reference exposes); ``bufs.value_offsets`` is the
raw device table.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def padded_stride(batch_size: int) -> int:
    return max(32, (int(batch_size) + 31) // 32 * 32)


@dataclass
class EvalBuffers:
    batch_size: int
    ldb: int
    xT: object           # int32 [num_vars x ldb]
    values_full: object  # fp32 [num_value_slots x ldb]
    scratch_full: object
    flows_full: object
    flow_scratch_full: object
    prod_flows_full: object
    f_params: object     # fp32 [f_params_size]
    lroot: object        # fp32 [B]
    work: object = None  # fp32 kernel workspace (block maxima), pcb_plan_workspace_floats
    batch: np.ndarray | None = None
    forward_done: bool = False
    backward_done: bool = False
    device: object = None
    _extra: dict = field(default_factory=dict)

    @property
    def value_offsets(self):
        return self.values_full[:, : self.batch_size]

    @property
    def values(self):
        """Node log values [slots x B] (offset + block base, materialised)."""
        import torch
        raw = self.values_full[:, : self.batch_size]
        vb = self._extra.get("slot_vb")
        n_sb = int(self._extra.get("n_sb_tot", 0))
        if vb is None or n_sb == 0:
            return raw
        base = self.work[: n_sb * self.ldb].view(n_sb, self.ldb)[:, : self.batch_size]
        add = base[vb.clamp(min=0)]
        return raw + torch.where((vb >= 0)[:, None], add, torch.zeros_like(add))

    @property
    def scratch(self):
        return self.scratch_full[:, : self.batch_size]

    @property
    def flows(self):
        return self.flows_full[:, : self.batch_size]

    @property
    def flow_scratch(self):
        return self.flow_scratch_full[:, : self.batch_size]

    @property
    def prod_flows(self):
        return self.prod_flows_full[:, : self.batch_size]


def allocate_buffers(compiled, batch_size: int, device=None, *, plan=None,
                     prod_flows: bool = True) -> EvalBuffers:
    """Zeroed device workspace for ``batch_size`` samples.  ``prod_flows=False``
    (training steps on plans whose product rows are each accumulated and
    pushed in one layer) leaves the product-flow table out: nothing reads it."""
    import torch
    from . import _lib
    from .plan import device_plan
    if plan is None:
        plan = device_plan(compiled, device)
    dev = plan.device
    b = int(batch_size)
    ldb = padded_stride(b)
    n_work = int(_lib.load().pcb_plan_workspace_floats(plan.handle, ldb))

    def z(rows):
        return torch.zeros((max(int(rows), 1), ldb), dtype=torch.float32, device=dev)

    slot_vb = plan.info["slot_vb"][: max(compiled.num_value_slots, 1)]
    bufs = EvalBuffers(
        batch_size=b, ldb=ldb,
        xT=torch.zeros((max(compiled.num_vars, 1), ldb), dtype=torch.int32, device=dev),
        values_full=z(compiled.num_value_slots),
        scratch_full=z(plan.info["scratch_rows"]),  # every layer's window stays resident
        flows_full=z(compiled.num_value_slots),
        flow_scratch_full=z(compiled.scratch_size),
        prod_flows_full=z(compiled.num_prod_rows) if prod_flows else z(0),
        f_params=torch.zeros(max(compiled.f_params_size, 1), dtype=torch.float32, device=dev),
        lroot=torch.zeros(max(b, 1), dtype=torch.float32, device=dev)[:b],
        work=torch.zeros(max(n_work, 1), dtype=torch.float32, device=dev),
        device=dev,
    )
    bufs._extra["slot_vb"] = torch.from_numpy(np.asarray(slot_vb, dtype=np.int64)).to(dev)
    bufs._extra["n_sb_tot"] = int(slot_vb.max()) + 1 if slot_vb.size else 0
    return bufs
