"""End-to-end SD engine on the tiny config (BASELINE config #1) with a real
offload budget, checked against the oracles at every layer boundary:

* routing indices of every captured verify layer = oracle router on the
  GPU's own layer input (bit-exact);
* the verify-MoE layer output = oracle experts + combine on that input,
  reading the expert blobs from the host pool rows (bit-exact);
* predicted expert sets, prefetched / demand-loaded transfers, final LRU
  order and slot assignment = the policy oracle replaying the recorded
  predictor outputs and verify routing in program order (exact);
* accepted lengths and correction tokens = oracle greedy acceptance on the
  GPU's verify logits (exact);
* SimReport accounting invariants of the reference (test_simcore.py:34-62).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def bits(t):
    if t.dtype == torch.bfloat16:
        return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return t.contiguous().cpu().numpy()


def make_engine(policy_kind="draft_prefetch", capacity=12, cutoff=3, N=4, batch=1, worker=True, record=True,
                capture=(0, 3), arch="tiny", ffn_impl="cuda_core", **kw):
    from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec, ProfiledTimings
    from paper_2510_10302_b200.engine import SpecMoEEngine
    from paper_2510_10302_b200.model import get_arch

    a = get_arch(arch)
    hw = HardwareSpec(gpu_memory=180_000_000_000, peak_non_expert_memory=8_000_000_000, pcie_bandwidth=55e9)
    t = ProfiledTimings(t_comp_target=1e-4, t_comp_draft=1e-4, t_io_expert=a.expert_bytes / 55e9)
    pol = PolicySpec(policy=Policy(policy_kind), prefetch_k=1, draft_length=N, acceptance_rate=1.0, seed=1234,
                     cutoff_layer=cutoff, cache_capacity_experts=capacity, worker_prefetch=worker)
    return SpecMoEEngine(a, hw, t, pol, batch=batch, record=record, capture_layers=capture, ffn_impl=ffn_impl, **kw)


def host_raw(eng, oracle, row):
    """Raw bf16 bits of a host-pool row, independently of the GPU decoder:
    the row itself (raw tier) or the CPU oracle's decode of its XC blob."""
    hp = eng.host_pool
    return hp.array[row] if hp.codec is None else oracle.xc_decode(hp.row_bytes(row))


def prompts(batch, P=12, vocab=512, seed=0):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (batch, P), generator=g)


def check_layer_captures(eng, oracle, tol=None):
    a = eng.arch
    n = 0
    for cap in eng.captures:
        if "layer" not in cap:
            continue
        l = cap["layer"]
        xn = bits(cap["xn"])
        w_o, idx_o, _, sg_o = oracle.router_topk(xn, bits(eng.weights.layers[l].router), a.top_k, a.renorm)
        assert np.array_equal(bits(cap["idx"]), idx_o), f"routing mismatch at layer {l}"
        assert np.array_equal(bits(cap["w"]).view(np.uint32), w_o.view(np.uint32))
        off, perm, inv = oracle.moe_permute(idx_o, a.num_experts)
        blobs = [host_raw(eng, oracle, eng.host_pool.row_of(l, e)) for e in range(a.num_experts)]
        _, y = oracle.expert_ffn(blobs, xn, a.ffn, off, perm)
        out = oracle.moe_combine(y, inv, w_o, xn.shape[0], a.hidden, a.top_k, residual=bits(cap["resid"]))
        if tol is None:
            assert np.array_equal(bits(cap["out"]), out), f"verify-MoE output mismatch at layer {l}"
        else:
            got = oracle.bf16_bits_to_f32(bits(cap["out"]))
            ref = oracle.bf16_bits_to_f32(out)
            assert np.abs(got - ref).max() <= tol * np.abs(ref).max(), f"verify-MoE output off at layer {l}"
        n += 1
    assert n > 0


def check_acceptance(eng, oracle):
    n = 0
    for cap in eng.captures:
        if "accept_logits" not in cap:
            continue
        am, res = oracle.greedy_accept(bits(cap["accept_logits"]), bits(cap["draft"]))
        assert np.array_equal(bits(cap["res"]), res)
        n += 1
    assert n > 0


def check_policy_replay(eng, state0):
    from oracle.policy_oracle import PrefetchReplay

    rep = PrefetchReplay(eng.capacity)
    order0, slots0 = state0
    rep.c.order = [tuple(e) for e in order0]
    rep.c.slot = {tuple(e): s for e, s in zip(order0, slots0)}
    rep.c.free = sorted(set(range(eng.capacity)) - set(slots0))
    for kind, layer, ids in eng.decisions:
        if kind == "task":
            rep.task(layer, ids)
        else:
            rep.verify(layer, ids)
    log = eng.cache.transfer_log()
    got = [(r["kind"], r["layer"], list(r["experts"])) for r in log]
    want = [(k, l, e) for (k, l, e, _) in rep.transfers]
    assert got == want
    assert [tuple(e) for e in eng.cache.lru_order] == rep.c.order
    for e in rep.c.order:
        assert eng.cache.slot_of(*e) == rep.c.slot[e]
    c = eng.cache.counters()
    assert (c["hits"], c["misses"]) == (rep.c.hits, rep.c.misses)
    assert c["prefetch_insertions"] == rep.c.prefetch_insertions
    assert c["prefetch_evictions"] == rep.c.prefetch_evictions
    assert c["demand_insertions"] == rep.c.demand_insertions
    assert c["tasks_completed"] == rep.tasks_completed


def run_and_check(oracle, tol=None, **kw):
    eng = make_engine(**kw)
    try:
        eng.prefill(prompts(eng.batch))
        state0 = ([tuple(e) for e in eng.cache.lru_order], [eng.cache.slot_of(*e) for e in eng.cache.lru_order])
        remaining = [20] * eng.batch
        while any(r > 0 for r in remaining):
            em = eng.step(remaining)
            remaining = [r - e for r, e in zip(remaining, em)]
        torch.cuda.synchronize()
        rep = eng.report()
        check_layer_captures(eng, oracle, tol)
        check_acceptance(eng, oracle)
        check_policy_replay(eng, state0)
        # reference accounting invariants (test_simcore.py:34-62)
        lookups = sum(len(set(ids)) for k, _, ids in eng.decisions if k == "verify")
        assert rep.counters["hits"] + rep.counters["misses"] == lookups
        for it in rep.iterations:
            assert 0 <= it.emitted <= it.accepted + 1 <= it.drafted + 1
        assert rep.emitted_tokens == 20 * eng.batch
        assert abs(sum(rep.latency_breakdown.values()) - 1.0) < 1e-6
        return eng, rep
    except Exception:
        eng.close()
        raise


def test_engine_tiny_draft_prefetch(oracle):
    eng, rep = run_and_check(oracle)
    try:
        assert rep.counters["prefetch_insertions"] > 0  # SP-MoE prefetch actually ran
        assert rep.counters["demand_insertions"] > 0  # offload is real (12 of 32 slots)
        assert rep.extras["acceptance_rate"] > 0.0
        assert rep.cutoff_effective == 3
    finally:
        eng.close()


@pytest.mark.parametrize("policy", ["on_demand", "gating_next_layer", "coarse_history"])
def test_engine_tiny_baseline_policies(oracle, policy):
    eng, rep = run_and_check(oracle, policy_kind=policy, cutoff=None)
    try:
        if policy == "on_demand":
            assert rep.counters["prefetch_insertions"] == 0
    finally:
        eng.close()


def test_engine_tiny_vanilla_executor(oracle):
    eng, rep = run_and_check(oracle, worker=False)
    eng.close()


def test_engine_tiny_batch4(oracle):
    eng, rep = run_and_check(oracle, batch=4)
    eng.close()


@pytest.mark.parametrize("ffn_impl", ["cuda_core", "auto"])
def test_engine_deterministic(oracle, ffn_impl):
    """Same seeds -> same tokens, same transfers, same cache counters (the
    worker thread's timing must not leak into any decision)."""
    outs = []
    for _ in range(2):
        eng = make_engine(record=False, capture=(), ffn_impl=ffn_impl)
        try:
            eng.prefill(prompts(1))
            for _ in range(4):
                eng.step()
            log = [(r["kind"], r["layer"], r["experts"]) for r in eng.cache.transfer_log()]
            outs.append((list(eng.seqs[0]), eng.cache.counters(), log))
        finally:
            eng.close()
    assert outs[0][0] == outs[1][0], "tokens differ"
    assert outs[0][2] == outs[1][2], "transfer sequence differs"
    assert outs[0][1] == outs[1][1], "cache counters differ"


def test_recalibrate_solver_and_measured_fallback():
    """engine.recalibrate: a feasible latency model sets the cutoff by the
    solver; one where even L = 0 misses the drafting window probes L = 0 and
    keeps it when its prefetch copies are hidden (tiny experts: they always
    are), or falls back to no prefetch with probing disabled.  The token
    stream is independent of all of it (caching never changes the math)."""
    from paper_2510_10302_b200 import ProfiledTimings

    ref = make_engine(record=False, capture=())
    try:
        ref.prefill(prompts(1))
        for _ in range(8):
            ref.step()
        want = list(ref.seqs[0])
    finally:
        ref.close()
    slow_link = ProfiledTimings(t_comp_target=1e-4, t_comp_draft=1e-6, t_io_expert=10.0)
    fast_link = ProfiledTimings(t_comp_target=1e-4, t_comp_draft=1e-2, t_io_expert=1e-6)
    for probe_steps in (2, 0):
        eng = make_engine(cutoff=None, capture=())
        try:
            eng.prefill(prompts(1))
            for _ in range(2):
                eng.step()
            assert eng.cutoff is not None
            eng.recalibrate(timings=fast_link, probe_steps=probe_steps)
            assert eng.cutoff_source == "solver" and eng.cutoff is not None and eng.cutoff >= 0
            eng.recalibrate(timings=slow_link, probe_steps=probe_steps)
            if probe_steps:
                assert eng.cutoff == 0 and eng.cutoff_source.startswith("measured"), eng.cutoff_source
            else:
                assert eng.cutoff is None and eng.cutoff_source == "solver"
            while len(eng.seqs[0]) < len(want):
                eng.step()
            torch.cuda.synchronize()
            assert list(eng.seqs[0])[: len(want)] == want
        finally:
            eng.close()


@pytest.mark.parametrize("tc_min", [2, 3])
def test_engine_tokens_independent_of_launch_grouping(oracle, tc_min):
    """Which resident experts share a K3 launch depends on copy timing
    (ready vs late slots); each expert's kernel path and split plan depend
    only on its own token count, so forcing every expert into its own launch
    gives the same tokens and the same verify-MoE bits."""
    outs = []
    for force_late in (False, True):
        eng = make_engine(capture=(0, 1, 2, 3), ffn_impl="auto", batch=3, tc_min_tokens=tc_min)
        try:
            eng.force_late = force_late
            eng.prefill(prompts(3))
            for _ in range(4):
                eng.step()
            torch.cuda.synchronize()
            caps = [bits(c["out"]) for c in eng.captures if "layer" in c]
            outs.append(([list(sq) for sq in eng.seqs], caps))
        finally:
            eng.close()
    assert outs[0][0] == outs[1][0], "tokens depend on launch grouping"
    assert len(outs[0][1]) == len(outs[1][1])
    assert all(np.array_equal(a, b) for a, b in zip(outs[0][1], outs[1][1]))


def test_flag_handoff_push_task():
    """push_task_flag: the worker waits for a device-bumped counter in mapped
    memory before reading the predicted ids (graph-safe hand-off)."""
    import ctypes as C

    from paper_2510_10302_b200 import _native
    from paper_2510_10302_b200.cache import NativeExpertCache

    lib = _native.load()
    host, dev = C.c_void_p(), C.c_void_p()
    _native.check("alloc", lib.spmoe_host_alloc_mapped(64, C.byref(host), C.byref(dev)))
    arr = (C.c_int32 * 16).from_address(host.value)
    arr[0], arr[1], arr[8] = 3, 5, 0  # ids at [0:2], counter at [8]
    pool = torch.empty((4, 64), dtype=torch.bfloat16, device="cuda")
    hostpool = torch.zeros((16, 64), dtype=torch.bfloat16).pin_memory()
    cs = torch.cuda.Stream()
    cache = NativeExpertCache(4, 2, 8, dev_pool_ptr=pool.data_ptr(), host_pool_ptr=hostpool.data_ptr(),
                              slot_bytes=128, copy_stream_ptr=cs.cuda_stream)
    try:
        cache.start_worker()
        _native.check("push", lib.spmoe_rt_push_task_flag(cache._h, 1, host.value, 2, host.value + 32, 1, 0))
        torch.cuda._sleep(20_000_000)  # the bump lands well after the push
        _native.check("bump", lib.spmoe_signal_bump(dev.value + 32, torch.cuda.current_stream().cuda_stream))
        cache.drain()
        assert arr[8] == 1
        assert cache.lookup((1, 3), False) and cache.lookup((1, 5), False)
    finally:
        cache.close()
        lib.spmoe_host_free(host)


def test_engine_shared_expert_arch(oracle):
    """DeepSeek/Qwen-style routing (no renorm, shared expert with sigmoid gate)
    at tiny width: routing and combine still bit-exact."""
    from paper_2510_10302_b200.model import ArchSpec, ARCH_PRESETS
    from dataclasses import replace

    a = replace(ARCH_PRESETS["tiny"], name="tiny_qwen", num_experts=16, top_k=4, renorm=False, shared_ffn=1024,
                shared_gate=True)
    import paper_2510_10302_b200.model as M

    M.ARCH_PRESETS["tiny_qwen"] = a
    eng = make_engine(arch="tiny_qwen", capacity=24, capture=(1,))
    try:
        eng.prefill(prompts(1))
        for _ in range(3):
            eng.step()
        torch.cuda.synchronize()
        for cap in eng.captures:
            if "layer" not in cap:
                continue
            l = cap["layer"]
            xn = bits(cap["xn"])
            lw = eng.weights.layers[l]
            w_o, idx_o, _, sg_o = oracle.router_topk(xn, bits(lw.router), a.top_k, a.renorm, bits(lw.shared_gate))
            assert np.array_equal(bits(cap["idx"]), idx_o)
            off, perm, inv = oracle.moe_permute(idx_o, a.num_experts)
            blobs = [host_raw(eng, oracle, eng.host_pool.row_of(l, e)) for e in range(a.num_experts)]
            _, y = oracle.expert_ffn(blobs, xn, a.ffn, off, perm)
            T = xn.shape[0]
            _, ys = oracle.expert_ffn([bits(lw.shared[0])], xn, a.shared_ffn, np.array([0, T], np.int32),
                                      np.arange(T, dtype=np.int32))
            out = oracle.moe_combine(y, inv, w_o, T, a.hidden, a.top_k, ys=ys[:T], sg=sg_o, residual=bits(cap["resid"]))
            assert np.array_equal(bits(cap["out"]), out)
    finally:
        eng.close()


def test_engine_tiny_tcgen05_path(oracle):
    """The default engine path (tcgen05 K3 for multi-token experts): routing,
    acceptance and the policy replay stay exact; the verify-MoE output
    matches the oracle within bf16 output rounding (2^-7 relative to the
    layer's max |value|, i.e. one bf16 ulp at the top of the range)."""
    eng, rep = run_and_check(oracle, tol=2.0 ** -7, ffn_impl="tcgen05", batch=2)
    eng.close()


def test_engine_trace_export_and_measured_timings(tmp_path):
    """§8(f) rows: real gating scores exported as trace-v1 (one row block
    per committed token), ProfiledTimings measured on the live engine."""
    from paper_2510_10302_b200.calibrate import measure_timings
    from paper_2510_10302_b200.tracefile import read_trace

    eng = make_engine(record=False, capture=(), record_routing=True)
    try:
        eng.prefill(prompts(1))
        remaining = [12]
        while remaining[0] > 0:
            remaining = [remaining[0] - eng.step(remaining)[0]]
        rep = eng.report()
        n = eng.export_trace(tmp_path / "trace.txt")
        fields, scores = read_trace(tmp_path / "trace.txt")
        assert n == rep.emitted_tokens == scores.shape[0]
        assert scores.shape[1:] == (eng.arch.num_layers, eng.arch.num_experts)
        assert np.allclose(scores.sum(-1), 1.0)
        t = measure_timings(eng)
        assert t.t_comp_draft > 0 and t.t_comp_target > 0 and t.t_io_expert > 0
    finally:
        eng.close()


def test_engine_timeline_csvs(tmp_path):
    """§8(f) row 3: SimReport CSV, transfers.csv and compute_slots.csv in the
    reference schema (report.py:22-23) from a real run, on one clock."""
    from paper_2510_10302_b200.report import (
        SLOTS_HEADER, TRANSFERS_HEADER, SimReport, write_compute_slots_csv, write_report_csv, write_transfer_log_csv)

    eng = make_engine(record=False, capture=(), record_timeline=True)
    try:
        eng.prefill(prompts(1))
        for _ in range(3):
            eng.step()
        rep = eng.report()
        L = eng.arch.num_layers
        assert sum(1 for s in rep.compute_slots if s.kind == "verify") == 3 * L
        assert sum(1 for s in rep.compute_slots if s.kind == "draft") == 3 * eng.policy.draft_length
        assert all(s.end >= s.start >= 0 for s in rep.compute_slots)
        write_compute_slots_csv(rep, tmp_path / "slots.csv")
        write_transfer_log_csv(rep, tmp_path / "transfers.csv")
        write_report_csv([rep], tmp_path / "report.csv")
        assert (tmp_path / "slots.csv").read_text().splitlines()[0] == SLOTS_HEADER
        assert (tmp_path / "transfers.csv").read_text().splitlines()[0] == TRANSFERS_HEADER
        rows = (tmp_path / "report.csv").read_text().splitlines()
        assert rows[0] == SimReport.csv_header() and len(rows) == 2
    finally:
        eng.close()


def test_failed_copy_is_reported_and_rolled_back():
    """A copy that cannot be issued (fault injection: the runtime's next
    copies fail as a rejected cudaMemcpyAsync would) surfaces as an error from the demand load and from the
    worker's drain, and never leaves the expert marked resident (SURVEY §5:
    copy errors surface as status codes)."""
    import numpy as np

    from paper_2510_10302_b200 import _native
    from paper_2510_10302_b200._native import SpmoeError
    from paper_2510_10302_b200.cache import ExpertId, NativeExpertCache

    lib = _native.load()
    pool = torch.empty((4, 64), dtype=torch.bfloat16, device="cuda")
    hostpool = torch.zeros((16, 64), dtype=torch.bfloat16).pin_memory()
    cs = torch.cuda.Stream()
    cache = NativeExpertCache(4, 2, 8, dev_pool_ptr=pool.data_ptr(), host_pool_ptr=hostpool.data_ptr(),
                              slot_bytes=128, copy_stream_ptr=cs.cuda_stream)
    try:
        _native.check("inject", lib.spmoe_rt_debug_fail_copies(cache._h, 1))
        with pytest.raises(SpmoeError):
            cache.demand_load([(0, 1), (0, 2)])
        assert ExpertId(0, 1) not in cache and ExpertId(0, 2) not in cache and len(cache) == 0
        cache.drain()  # the demand error was already returned
        cache.demand_load([(0, 1)])  # the runtime keeps working
        cache.drain()
        assert ExpertId(0, 1) in cache
        _native.check("inject", lib.spmoe_rt_debug_fail_copies(cache._h, 1))
        cache.start_worker()
        idx = np.array([4], np.int32)
        ev = torch.cuda.Event()
        ev.record()
        _native.check("push", lib.spmoe_rt_push_task(cache._h, 1, idx.ctypes.data, 1, ev.cuda_event, 0))
        with pytest.raises(SpmoeError):
            cache.drain()
        assert ExpertId(1, 4) not in cache
        assert cache.counters()["tasks_aborted"] == 1
    finally:
        cache.close()
