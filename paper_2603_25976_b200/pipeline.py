"""Host -> device input pipeline for training loops over host-resident data.

`BatchPrefetcher` keeps two device slots per input and copies batch k+1 from pinned host
memory on its own copy stream while step k runs, so the PCIe transfer of a step's inputs
overlaps the previous step's kernels instead of preceding its own.  The compute stream
waits on the copy's event before the step reads the slot (stream order, no host sync);
a slot is overwritten only after every kernel enqueued before the batch that used it
(a copy-stream wait on an event recorded when the slot was handed out).

The reference's batcher (harness/run.py:174-192) yields host arrays that the step
consumes synchronously; here the same batches arrive device-resident.
"""

from __future__ import annotations

import numpy as np
import torch

from .models import Batch
from .runtime import runtime


def _pinned(a, dtype):
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    t = t.to(dtype) if t.dtype != dtype else t
    return t if t.is_pinned() else t.contiguous().pin_memory()


class BatchPrefetcher:
    """Yields device `Batch`es from a host source, one batch ahead.

    source: an iterator (or callable returning the next item) of (X, y) pairs (numpy or
    torch, pinned or not; unpinned inputs are pinned once per batch) or host `Batch`es.
    loss_kind: "ce" (y int64 class indices) or "mse" (y float targets)."""

    def __init__(self, source, loss_kind: str, global_size: int | None = None, row_offset: int = 0, device=None):
        self._next_item = source if callable(source) else iter(source).__next__
        self.loss_kind = loss_kind
        self.global_size = global_size
        self.row_offset = row_offset
        self.device = device if device is not None else runtime().device
        self.copy_stream = torch.cuda.Stream(self.device)
        self._slots = [None, None]
        self._ready = [None, None]   # copy-complete events
        self._free = [None, None]    # slot released (compute stream) events
        self._pending = None         # slot index holding the prefetched batch
        self.h2d_bytes = 0           # bytes of the last batch copied

    def _host_pair(self):
        item = self._next_item()
        if isinstance(item, Batch):
            X, y = item.inputs, item.targets
        else:
            X, y = item
        ydt = torch.int64 if self.loss_kind == "ce" else torch.float32
        return _pinned(X, torch.float32), _pinned(y, ydt)

    def _issue(self, i):
        Xh, yh = self._host_pair()
        slot = self._slots[i]
        if slot is None or slot[0].shape != Xh.shape or slot[1].shape != yh.shape:
            slot = (torch.empty(Xh.shape, dtype=torch.float32, device=self.device),
                    torch.empty(yh.shape, dtype=yh.dtype, device=self.device))
            self._slots[i] = slot
        cs = self.copy_stream
        if self._free[i] is not None:
            cs.wait_event(self._free[i])
        with torch.cuda.stream(cs):
            slot[0].copy_(Xh, non_blocking=True)
            slot[1].copy_(yh, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        # the pinned host buffers must outlive the copies: keep them with the slot
        self._ready[i] = (ev, Xh, yh)
        self.h2d_bytes = Xh.numel() * Xh.element_size() + yh.numel() * yh.element_size()

    def next(self) -> Batch:
        if self._pending is None:
            self._issue(0)
            self._pending = 0
        i = self._pending
        compute = torch.cuda.current_stream(self.device)
        compute.wait_event(self._ready[i][0])
        X, y = self._slots[i]
        # label-range contract from the host copy: no device read (no sync) per batch
        hint = {}
        if self.loss_kind == "ce":
            yh = self._ready[i][2]
            hint = {"_ymin": int(yh.min()), "_ymax": int(yh.max())}
        batch = Batch(X, y, self.loss_kind, global_size=self.global_size, row_offset=self.row_offset, _dev=hint)
        # the other slot held the previous batch: reusable once the work enqueued so far is done
        j = 1 - i
        ev = torch.cuda.Event()
        ev.record(compute)
        self._free[j] = ev
        self._issue(j)
        self._pending = j
        return batch

    __next__ = next

    def __iter__(self):
        return self
