"""Expert-parallel verify MoE on one B200: the row-gather kernel against
torch indexing, and the EP engine (world size 1 without a process group,
and over a one-rank NCCL group so the all-to-all path runs) against the
oracle at captured layer boundaries and against the non-EP engine token
for token, with the on_demand and the draft_prefetch policy."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from test_engine_gpu import bits, check_acceptance, check_layer_captures, make_engine, prompts

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,shape,div", [
    (torch.bfloat16, (40, 4096), 2),
    (torch.float32, (33, 2048), 1),
    (torch.bfloat16, (17, 6), 3),  # 12-byte rows: 4-byte word path
    (torch.int32, (50,), 1),
])
def test_gather_rows(native, dtype, shape, div):
    from paper_2510_10302_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(7)
    src = torch.randint(-1000, 1000, shape, generator=g, device="cuda").to(dtype)
    n = shape[0] * div + 5
    idx = torch.randint(0, shape[0] * div, (n,), generator=g, device="cuda", dtype=torch.int32)
    out = K.gather_rows(src, idx, div)
    torch.cuda.synchronize()
    ref = src[idx.long() // div]
    assert torch.equal(out, ref)
    assert K.gather_rows(src, idx[:0], div).shape[0] == 0


def _run(eng, steps=4):
    eng.prefill(prompts(eng.batch))
    out = []
    for _ in range(steps):
        out.append(eng.step())
    torch.cuda.synchronize()
    return out, [list(s) for s in eng.seqs]


@pytest.mark.parametrize("batch", [1, 3])
def test_ep_engine_matches_local(oracle, batch):
    kw = dict(policy_kind="on_demand", cutoff=None, capacity=12, batch=batch, capture=(0, 2, 3))
    ep = make_engine(expert_parallel=True, **kw)
    try:
        assert ep.ep is not None and ep.ep.world == 1
        em_ep, seq_ep = _run(ep)
        check_layer_captures(ep, oracle)
        check_acceptance(ep, oracle)
        assert ep.ep.bytes_sent == 0
        assert ep.report().counters["demand_insertions"] > 0
    finally:
        ep.close()
    ref = make_engine(**kw)
    try:
        em_ref, seq_ref = _run(ref)
    finally:
        ref.close()
    assert em_ep == em_ref
    assert seq_ep == seq_ref


def test_ep_engine_rejects_other_prefetch_policies():
    from paper_2510_10302_b200.config import ValidationError

    for kind in ("gating_next_layer", "coarse_history"):
        with pytest.raises(ValidationError):
            make_engine(expert_parallel=True, policy_kind=kind, cutoff=None)


@pytest.mark.parametrize("batch", [1, 2])
def test_ep_engine_draft_prefetch_matches_local(oracle, batch):
    """EP with the draft_prefetch policy (ep.py: predictions gathered on the
    host, each rank enqueues the ones it owns): at world size 1 the owned
    union is the rank's own prediction, so tokens, cache decisions and
    counters equal the non-EP engine's (which hands the indices to the worker
    through mapped memory and event waits instead)."""
    kw = dict(policy_kind="draft_prefetch", cutoff=3, capacity=12, batch=batch, capture=(0, 3))
    ep = make_engine(expert_parallel=True, **kw)
    try:
        em_ep, seq_ep = _run(ep)
        check_layer_captures(ep, oracle)
        check_acceptance(ep, oracle)
        rep_ep = ep.report()
        xfer_ep = [(t.kind, t.layer, tuple(t.experts)) for t in ep.transfers()]
        tasks_ep = [(l, sorted(set(i for i in ids if i >= 0))) for kind, l, ids in ep.decisions if kind == "task"]
    finally:
        ep.close()
    ref = make_engine(**kw)
    try:
        em_ref, seq_ref = _run(ref)
        rep_ref = ref.report()
        xfer_ref = [(t.kind, t.layer, tuple(t.experts)) for t in ref.transfers()]
        tasks_ref = [(l, sorted(set(i for i in ids if i >= 0))) for kind, l, ids in ref.decisions if kind == "task"]
    finally:
        ref.close()
    assert em_ep == em_ref and seq_ep == seq_ref
    assert rep_ep.counters["prefetch_insertions"] == rep_ref.counters["prefetch_insertions"] > 0
    for key in ("hits", "misses", "demand_insertions", "evictions"):
        assert rep_ep.counters[key] == rep_ref.counters[key], key
    # the same prefetch tasks (EP drops the -1 padding and duplicates) and
    # the same copy batches (prefetch and demand), layers and experts, in order
    assert tasks_ep == [t for t in tasks_ref if t[1]]
    assert xfer_ep == xfer_ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("policy_kind,cutoff", [("on_demand", None), ("draft_prefetch", 3)])
def test_ep_engine_nccl_group_of_one(oracle, policy_kind, cutoff):
    """The all-to-all path over a real (one-rank) NCCL group; with
    draft_prefetch also the host-side prediction exchange and the cutoff
    agreement over the gloo group the exchange creates beside it."""
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        eng = make_engine(expert_parallel=True, policy_kind=policy_kind, cutoff=cutoff, capacity=16, capture=(1,))
        try:
            assert not eng.ep.local_only and eng.ep.host_group is not None
            _run(eng, steps=3)
            check_layer_captures(eng, oracle)
            check_acceptance(eng, oracle)
            if policy_kind == "draft_prefetch":
                assert eng.cutoff == cutoff and eng.report().counters["prefetch_insertions"] > 0
        finally:
            eng.close()
    finally:
        dist.destroy_process_group()
