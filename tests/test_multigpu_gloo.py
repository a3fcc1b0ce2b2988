"""N>1 host logic on CPU: world_size 2 over gloo (127.0.0.1).  Covers the
replica stream split, the max-over-ranks timing / summed-token reduction
bench.py uses, and the /dev/shm shared host expert pool (leader fills,
follower attaches and sees identical bytes)."""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_10302_b200.replicas import assign_streams


def test_assign_streams_partition():
    for n in range(0, 20):
        for world in range(1, 9):
            got = [assign_streams(n, r, world) for r in range(world)]
            flat = [s for g in got for s in g]
            assert flat == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shm_root, q):
    import torch.distributed as dist

    from paper_2510_10302_b200.replicas import SharedHostPool, reduce_run

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms, wall, tok = reduce_run(10.0 + rank, 1.0 + 2 * rank, 5 + rank)

        def fill(a):
            a[:] = np.arange(a.size, dtype=np.uint64).reshape(a.shape).astype(np.uint16)

        pool = SharedHostPool("gloo_test", rows=4, row_elems=1024, leader=(rank == 0), fill=fill, register=False,
                              root=shm_root, timeout_s=60)
        dist.barrier()
        checksum = int(pool.array.astype(np.uint64).sum())
        pool.close(unlink=False)
        dist.barrier()
        q.put((rank, ms, wall, tok, checksum))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduction_and_shared_pool():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as shm_root:
        procs = [ctx.Process(target=_worker, args=(r, world, port, shm_root, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = sorted(q.get(timeout=120) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    expect_sum = int((np.arange(4 * 1024, dtype=np.uint64).astype(np.uint16)).astype(np.uint64).sum())
    for rank, ms, wall, tok, checksum in res:
        assert ms == pytest.approx(11.0)  # max over ranks
        assert wall == pytest.approx(3.0)
        assert tok == 11  # sum over ranks
        assert checksum == expect_sum  # follower sees the leader's bytes


def test_numa_pool_roles_one_leader_per_node():
    from paper_2510_10302_b200.replicas import node_cpus, numa_pool_roles

    nodes = [0, 0, 0, 0, 1, 1, 1, 1]
    roles = [numa_pool_roles(nodes, r) for r in range(8)]
    assert [n for n, _ in roles] == nodes
    assert [r for r, (_, lead) in enumerate(roles) if lead] == [0, 4]
    # interleaved placement: the lowest local rank on each node leads
    assert [numa_pool_roles([1, 0, 1, 0], r)[1] for r in range(4)] == [True, True, False, False]
    assert numa_pool_roles([0], 0) == (0, True)
    assert len(node_cpus(0)) >= 1 and node_cpus(10_000) == []


def test_plan_host_pools_shared_private_and_bounded():
    from paper_2510_10302_b200.replicas import plan_host_pools

    GB = 10**9
    # two NUMA pools of 61 GB fit a 1 TB shm
    assert plan_host_pools(2, 61 * GB, 8, 256, 1000 * GB, 1500 * GB) == (True, None)
    # 64 GB docker shm: private pools, all 8 fit in 1.5 TB of RAM
    assert plan_host_pools(2, 61 * GB, 8, 256, 64 * GB, 1500 * GB) == (False, None)
    # small RAM: private pools with aliased rows so 8 x pool <= 80 % of RAM
    use, distinct = plan_host_pools(2, 61 * GB, 8, 256, 64 * GB, 200 * GB)
    assert not use and 1 <= distinct < 256
    assert 8 * distinct * (61 * GB // 256) <= 0.8 * 200 * GB
