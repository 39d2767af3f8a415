"""Batch sources for ``train()``: the training batches of one epoch, in
order, delivered into a step's static device input.

``DeviceBatches``: the dataset already resident on the device (validated
once there); a batch is one ``index_select`` into the step's input.

``HostBatches``: a host (numpy) dataset streamed to the device.  A loader
thread gathers each batch's rows in epoch order (the reference's
``data[order[a:a + bs]]``, ``pcirc/train.py:130``) into a ring of pinned
buffers and validates them (``engine.py:36-52``: a bad batch raises
``FormatError`` when its step is reached, after the steps before it, as the
reference's per-batch forward does); the host-to-device copy runs on a copy
stream into one of two device staging buffers while the previous step
computes, and the step takes its batch with one device-to-device copy.  The
gathers and copies overlap the GPU work, so an epoch from host data runs at
the device-resident rate.
"""
from __future__ import annotations

import queue
import threading

import numpy as np

from ..errors import FormatError


def check_rows(rows: np.ndarray, cats: np.ndarray) -> None:
    """Category checks of ``engine.py:36-52`` on a [B x vars] block."""
    if rows.size == 0:
        return
    if rows.min() < -1:
        raise FormatError("category values must be >= 0, or -1 for missing")
    bad = (rows >= cats[None, :]).any(axis=0)
    if bad.any():
        var = int(np.flatnonzero(bad)[0])
        raise FormatError(f"variable {var} has values outside [0, {int(cats[var])})")


class DeviceBatches:
    def __init__(self, data_dev, order_dev, spans):
        self.data, self.order, self.spans = data_dev, order_dev, spans

    def fill(self, i, dst):
        import torch
        a, b = self.spans[i]
        if b > a:
            torch.index_select(self.data, 0, self.order[a:b], out=dst[: b - a])

    def close(self):
        pass


class HostBatches:
    def __init__(self, data: np.ndarray, order: np.ndarray, spans, cats, dev, slots: int = 4):
        import torch
        self.spans = spans
        nv = data.shape[1]
        bmax = max([b - a for a, b in spans] + [1])
        self.slots = slots
        self.pinned = [torch.empty((bmax, nv), dtype=torch.int32).pin_memory()
                       for _ in range(slots)]
        self.pinned_np = [p.numpy() for p in self.pinned]
        self.stage = [torch.empty((bmax, nv), dtype=torch.int32, device=dev) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(dev)
        self.h2d_done = [torch.cuda.Event() for _ in range(slots)]
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.used = [torch.cuda.Event() for _ in range(2)]
        self.comp = torch.cuda.current_stream(dev)
        self.q: queue.Queue = queue.Queue()
        self.free = threading.Semaphore(slots)
        self.stop = False
        self.data, self.order, self.cats = data, order, np.asarray(cats)
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        d = self.data
        direct = d.dtype == np.int32
        for i, (a, b) in enumerate(self.spans):
            self.free.acquire()
            if self.stop:
                return
            slot = i % self.slots
            if i >= self.slots:
                self.h2d_done[slot].synchronize()  # the slot's last copy has left
            err = None
            try:
                buf = self.pinned_np[slot][: b - a]
                rows = self.order[a:b]
                if direct:
                    np.take(d, rows, axis=0, out=buf)
                    check_rows(buf, self.cats)
                else:
                    blk = d[rows]
                    check_rows(blk, self.cats)
                    buf[:] = blk
            except Exception as e:  # surfaced when the step is reached
                err = e
            self.q.put((slot, err))
            if err is not None:
                return

    def fill(self, i, dst):
        slot, err = self.q.get()
        if err is not None:
            self.close()
            raise err
        a, b = self.spans[i]
        k = i % 2
        cs = self.copy_stream
        if i >= 2:
            cs.wait_event(self.used[k])
        else:
            cs.wait_stream(self.comp)
        import torch
        with torch.cuda.stream(cs):
            if b > a:
                self.stage[k][: b - a].copy_(self.pinned[slot][: b - a], non_blocking=True)
            self.copied[k].record(cs)
            self.h2d_done[slot].record(cs)
        self.free.release()
        self.comp.wait_event(self.copied[k])
        if b > a:
            dst[: b - a].copy_(self.stage[k][: b - a], non_blocking=True)
        self.used[k].record(self.comp)

    def close(self):
        self.stop = True
        for _ in range(self.slots):
            self.free.release()
        self.thread.join(timeout=10)
