"""Critical-expert selection and the draft-guided predictor.

Drop-in names from moesim (``predictor.py:46-106``, ``trace.py:28-37``):
``top_k_indices``, ``select_critical``, ``CriticalExpertSet``,
``HistoryCounter``.  The reference's predictor is a fidelity knob mixing
ground-truth trace scores with noise; the B200 build replaces it with the
paper's predictor (Algorithm 1 l.2-3): the draft model's
layer-l MLP input is projected through the *target* layer-l router by the
fused K1 kernel, whose top-k indices land in mapped pinned memory for the
prefetch worker (:class:`DraftGuidedPredictor`).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np


def top_k_indices(scores: Sequence[float], k: int) -> tuple[int, ...]:
    """The k largest scores' indices, largest first, ties -> lowest index."""
    arr = np.asarray(scores)
    n = arr.shape[0]
    if k > n:
        raise ValueError(f"k={k} exceeds vector length {n}")
    # lexicographic key (-score, index): stable sort of the negated scores
    order = np.lexsort((np.arange(n), -arr))
    return tuple(int(i) for i in order[:k])


@dataclass(frozen=True)
class CriticalExpertSet:
    """Top-k predicted experts of one layer, descending score."""

    layer: int
    experts: tuple[int, ...]
    scores: tuple[float, ...]


def select_critical(scores: Sequence[float], k: int, layer: int = 0) -> CriticalExpertSet:
    arr = np.asarray(scores, dtype=float)
    if k > arr.shape[0]:
        raise ValueError(f"k={k} exceeds score vector length {arr.shape[0]}")
    return CriticalExpertSet(layer=layer, experts=top_k_indices(arr, k), scores=tuple(map(float, arr)))


class HistoryCounter:
    """Per-layer activation counts (coarse-history baseline policy)."""

    def __init__(self, num_layers: int, experts_per_layer: int):
        self.counts = np.zeros((num_layers, experts_per_layer), dtype=np.int64)

    def record(self, layer: int, experts: Sequence[int]) -> None:
        for e in experts:
            self.counts[layer, e] += 1

    def record_many(self, layer: int, experts: np.ndarray) -> None:
        np.add.at(self.counts[layer], np.asarray(experts, dtype=np.int64).ravel(), 1)

    def scores(self, layer: int) -> np.ndarray:
        row = self.counts[layer]
        total = row.sum()
        return np.full(row.shape[0], 1.0 / row.shape[0]) if total == 0 else row / total


class DraftGuidedPredictor:
    """Algorithm 1 on the GPU: ``Gates[l](s)`` + ``TopK_Index`` fused in K1.

    Owns a ring of mapped pinned int32 buffers (one entry per (draft step,
    layer) task of an iteration) and a matching ring of CUDA events; each
    :meth:`predict` launches K1 on the current stream writing the indices
    straight into the ring entry, records the entry's event and returns the
    (host pointer, device pointer, event) hand-off for the worker.
    """

    def __init__(self, entries: int, width: int):
        import ctypes as C

        import torch

        from . import _native

        self.entries = entries
        self.width = width  # ints per entry (batch * prefetch_k)
        lib = _native.load()
        host = C.c_void_p()
        dev = C.c_void_p()
        nbytes = max(entries * width * 4, 4)
        _native.check("spmoe_host_alloc_mapped", lib.spmoe_host_alloc_mapped(nbytes, C.byref(host), C.byref(dev)))
        self._lib = lib
        self.host_ptr = host.value
        self.dev_ptr = dev.value
        buf = (C.c_int32 * (entries * width)).from_address(self.host_ptr)
        self.view = np.ctypeslib.as_array(buf).reshape(entries, width)
        self.view[:] = -1
        # raw CUDA events (recorded as external event nodes when a draft step
        # is captured in a CUDA graph, so the worker can wait on them)
        self.events = []
        for _ in range(entries):
            ev = C.c_void_p()
            _native.check("spmoe_event_create", lib.spmoe_event_create(C.byref(ev)))
            self.events.append(ev.value)
        self.next = 0

    def reset(self) -> None:
        self.next = 0

    def entry(self) -> int:
        if self.next >= self.entries:
            raise RuntimeError("predictor ring exhausted (drain before reuse)")
        self.next += 1
        return self.next - 1

    def host_ptr_of(self, i: int) -> int:
        return self.host_ptr + 4 * i * self.width

    def predict_at(self, i: int, x_last, router_w, k: int, renorm: bool, weights_out, idx_out) -> None:
        """K1 on ``x_last`` [B, H] against the target router writing ring
        entry ``i``, then record entry i's event on the current stream."""
        import torch

        from . import _native
        from .kernels import router_topk

        dptr = self.dev_ptr + 4 * i * self.width
        router_topk(x_last, router_w, k, renorm, host_idx_dev_ptr=dptr, out=(weights_out, idx_out))
        _native.check(
            "spmoe_event_record_external",
            self._lib.spmoe_event_record_external(self.events[i], torch.cuda.current_stream().cuda_stream),
        )

    def predict(self, x_last, router_w, k: int, renorm: bool, weights_out, idx_out):
        """Eager form: next free entry; returns (index, host_ptr, event)."""
        i = self.entry()
        self.predict_at(i, x_last, router_w, k, renorm, weights_out, idx_out)
        return i, self.host_ptr_of(i), self.events[i]

    def close(self) -> None:
        import ctypes as C

        if getattr(self, "host_ptr", None):
            self.view = None
            for ev in self.events:
                self._lib.spmoe_event_destroy(ev)
            self.events = []
            self._lib.spmoe_host_free(C.c_void_p(self.host_ptr))
            self.host_ptr = None
