"""Multi-GPU replica plumbing (SURVEY.md §8 e): one process per GPU, each an
independent SD request stream with its own HBM slot pool, copy stream and
PCIe link.  There is no data-path collective; ranks only

* split the request streams (:func:`assign_streams`),
* agree on timing (max over ranks) and totals (sum) (:func:`reduce_run`),
* share ONE page-locked host expert pool per NUMA node through /dev/shm
  instead of pinning the pool per process (:class:`SharedHostPool`,
  :func:`numa_pool_roles`): each GPU reads experts from DRAM on its own
  socket, so 8 concurrent host links do not funnel through one socket's
  memory controllers and the inter-socket link.

All functions take a ``torch.distributed`` process group (NCCL on the GPU
box, gloo in the CPU tests).
"""

from __future__ import annotations

import mmap
import os
import time
from pathlib import Path

import numpy as np


def gpu_numa_node(device_index: int) -> int:
    """NUMA node of a GPU's PCIe root (sysfs); 0 when unknown (single-node
    hosts, containers without sysfs)."""
    try:
        import torch

        pr = torch.cuda.get_device_properties(device_index)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        v = int(Path(f"/sys/bus/pci/devices/{bus}/numa_node").read_text().strip())
        return max(v, 0)
    except Exception:
        return 0


def node_cpus(node: int) -> list[int]:
    """CPUs of a NUMA node (sysfs cpulist), [] if unknown."""
    try:
        text = Path(f"/sys/devices/system/node/node{node}/cpulist").read_text().strip()
    except OSError:
        return []
    cpus: list[int] = []
    for part in text.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.extend(range(int(a), int(b) + 1))
        elif part:
            cpus.append(int(part))
    return cpus


def numa_pool_roles(nodes: list[int], local_rank: int) -> tuple[int, bool]:
    """One shared host pool per NUMA node: ``nodes[r]`` = NUMA node of local
    rank r's GPU.  Returns (this rank's node, whether it leads (creates and
    fills) that node's pool: the lowest local rank on the node)."""
    node = nodes[local_rank]
    leader = min(r for r, n in enumerate(nodes) if n == node) == local_rank
    return node, leader


def bind_to_node(node: int) -> bool:
    """Run this process on its GPU's NUMA node, so the host pool pages it
    first-touches (and pins) are local to that socket.  False if unknown."""
    cpus = node_cpus(node)
    if not cpus:
        return False
    try:
        os.sched_setaffinity(0, cpus)
        return True
    except OSError:
        return False


def shm_free_bytes(root: str = "/dev/shm") -> int:
    """Free bytes of the shared-memory filesystem (0 if absent)."""
    try:
        st = os.statvfs(root)
        return st.f_bavail * st.f_frsize
    except OSError:
        return 0


def mem_available_bytes() -> int:
    """MemAvailable from /proc/meminfo (0 if unknown)."""
    try:
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def plan_host_pools(n_pools: int, pool_bytes: int, n_procs: int, rows: int, shm_free: int, mem_free: int,
                    headroom: float = 0.8) -> tuple[bool, int | None]:
    """How the ranks of one box hold the host expert tier.

    Shared /dev/shm pools (one per NUMA node) when they fit in ``headroom`` of
    the shm filesystem; otherwise one private pinned pool per process, with
    ``distinct`` rows (experts alias rows: bytes per copy unchanged) bounded
    so that all private pools fit in ``headroom`` of the available RAM.
    Returns (use_shared, distinct_rows or None)."""
    if n_pools * pool_bytes <= headroom * shm_free:
        return True, None
    per_row = max(1, pool_bytes // max(1, rows))
    budget = headroom * mem_free / max(1, n_procs) if mem_free else pool_bytes
    if pool_bytes <= budget:
        return False, None
    return False, max(1, int(budget // per_row))


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
