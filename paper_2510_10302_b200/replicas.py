"""Multi-GPU replica plumbing (SURVEY.md §8 e): one process per GPU, each an
independent SD request stream with its own HBM slot pool, copy stream and
PCIe link.  There is no data-path collective; ranks only

* split the request streams (:func:`assign_streams`),
* agree on timing (max over ranks) and totals (sum) (:func:`reduce_run`),
* share ONE page-locked host expert pool per box through /dev/shm instead of
  pinning L·E·expert_bytes per process (:class:`SharedHostPool`).

All functions take a ``torch.distributed`` process group (NCCL on the GPU
box, gloo in the CPU tests).
"""

from __future__ import annotations

import mmap
import os
import time
from pathlib import Path

import numpy as np


def assign_streams(n_streams: int, rank: int, world: int) -> list[int]:
    """Request-stream ids owned by ``rank``: contiguous, balanced to one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_streams, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def reduce_run(device_ms: float, wall_s: float, emitted: int, group=None, device=None) -> tuple[float, float, int]:
    """(max device ms, max wall s, total emitted tokens) over ranks.  Uses
    float64 so large token counts stay exact."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(device_ms), float(wall_s), int(emitted)
    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    mx = torch.tensor([device_ms, wall_s], dtype=torch.float64, device=dev)
    sm = torch.tensor([float(emitted)], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
    return float(mx[0]), float(mx[1]), int(round(float(sm[0])))


class SharedHostPool:
    """A /dev/shm-backed expert pool shared by the ranks of one box.

    The local leader (local rank 0) creates and fills the file, writes a
    ready marker, and every rank maps it (and, on a GPU box, page-locks its
    mapping with ``spmoe_host_register`` so copies run at the pinned peak).
    Followers wait for the marker.  ``fill(array)`` is called by the leader
    only.
    """

    def __init__(self, name: str, rows: int, row_elems: int, leader: bool, fill=None, timeout_s: float = 1800.0,
                 register: bool = True, root: str = "/dev/shm", publish: bool = True):
        self.path = Path(root) / f"spmoe_{name}.pool"
        self.ready = Path(root) / f"spmoe_{name}.ready"
        self.nbytes = rows * row_elems * 2
        self.rows, self.row_elems = rows, row_elems
        if leader:
            if self.ready.exists():
                self.ready.unlink()
            with open(self.path, "wb") as f:
                f.truncate(self.nbytes)
        else:
            t0 = time.time()
            while not self.ready.exists():
                if time.time() - t0 > timeout_s:
                    raise TimeoutError(f"shared host pool {self.path} never became ready")
                time.sleep(0.2)
        fd = os.open(self.path, os.O_RDWR)
        try:
            self._mm = mmap.mmap(fd, self.nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self.array = np.frombuffer(self._mm, dtype=np.uint16).reshape(rows, row_elems)
        self.ptr = self.array.ctypes.data
        self._registered = False
        self.leader = leader
        if leader:
            if fill is not None:
                fill(self.array)
            if publish:
                self.publish()
        if register:
            from . import _native

            lib = _native.load()
            _native.check("spmoe_host_register", lib.spmoe_host_register(self.ptr, self.nbytes))
            self._registered = True

    def publish(self) -> None:
        """Leader: the pool content is complete; unblock the followers."""
        self._mm.flush()
        self.ready.write_text(str(os.getpid()))

    def close(self, unlink: bool = False) -> None:
        if self._registered:
            from . import _native

            _native.load().spmoe_host_unregister(self.ptr)
            self._registered = False
        self.array = None
        try:
            self._mm.close()
        except (BufferError, ValueError):
            pass
        if unlink:
            for p in (self.path, self.ready):
                try:
                    p.unlink()
                except FileNotFoundError:
                    pass
