"""The real draft/verify decode loop on one B200 (replaces moesim.simcore).

One :class:`SpecMoEEngine` owns, for B independent sequences on one GPU:

* the HBM slot pool ``[capacity, 3*F*H]`` and the native slot-table runtime
  (LRU metadata, copy stream, per-slot events, prefetch worker thread);
* the pinned host expert pool (the offload tier);
* target and draft KV caches and the deterministic random weights.

Per iteration (``Simulation.run`` of ``simcore.py:426-465``):

1. drafting (``_draft_stage`` ``simcore.py:323-354``): N draft steps; at every
   draft layer l <= cutoff the draft's MLP input is projected through the
   *target* router l by K1, whose indices land in mapped pinned memory; an
   event is recorded and the task is pushed to the worker thread
   (Algorithm 1), which waits on the event, filters resident experts, picks
   LRU victims and issues batched H2D copies on the copy stream
   (Algorithm 2).  The draft token chain stays on the device.
2. verification (``_verify_stage`` ``simcore.py:356-422``) of the N+1 tokens
   ``[last committed, d_0..d_{N-1}]``: per layer, K1 routes on the GPU, the
   host reads the indices (zero-copy), touches the union of required experts
   in ascending order, demand-loads the misses behind queued prefetches
   (``on_demand_load``), then runs K2 permute, K3 for cache-resident experts
   first and for each late expert after its slot's ready event (PAPER.md
   §4.3 cached-first order), and K4 combine + residual.
3. K6 greedy acceptance: longest matching prefix + correction/bonus token;
   KV caches roll back by length bookkeeping.

Accounting follows ``SimReport`` (``simcore.py:79-170,467-502``) with device
times from CUDA events: ``expert_load`` is the time the compute stream sat in
``cudaStreamWaitEvent`` on slot copies, ``draft`` the drafting span,
``attention_and_other`` the rest of verification.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import kernels as K
from .cache import ExpertId, NativeExpertCache
from .config import HardwareSpec, Policy, PolicySpec, ProfiledTimings, ValidationError, cache_capacity_slots
from .cutoff import cutoff_input_from_specs, solve_cutoff
from .model import ArchSpec, HostExpertPool, KVCache, attention_block, build_weights, lm_logits, model_spec_for, rms_norm
from .predictor import DraftGuidedPredictor, HistoryCounter, top_k_indices
from .report import ComputeSlot, IterationRecord, SimReport, TransferKind, TransferRecord


def effective_cutoff(model, hw, timings, policy, window_tokens: int = 1, k_eff: int | None = None) -> int | None:
    """Cutoff honoured by the engine: explicit override, else the solver's
    answer (None = infeasible -> no drafting-stage prefetch), clamped to both
    depths (``simcore.py:182-197``).  ``k_eff`` replaces prefetch_k as the
    per-layer expert count (measured distinct prefetches per layer over an
    N-token window, see :meth:`SpecMoEEngine.recalibrate`)."""
    if policy.cutoff_layer is not None:
        layer = policy.cutoff_layer
    else:
        k = max(policy.prefetch_k, k_eff or 0)
        res = solve_cutoff(cutoff_input_from_specs(model, hw, timings, k, window_tokens=window_tokens))
        if not res.feasible:
            return None
        layer = res.layer
    return min(layer, model.draft_layers - 1, model.num_layers - 1)


@dataclass
class _Stall:
    kind: str  # "prefetch" (waited on an in-flight prefetch) | "demand"
    layer: int
    a: torch.cuda.Event
    b: torch.cuda.Event


class _Scratch:
    """Preallocated per-layer MoE buffers for up to ``T`` tokens."""

    def __init__(self, arch: ArchSpec, T: int, device):
        H, k = arch.hidden, arch.top_k
        f32, i32, bf = torch.float32, torch.int32, torch.bfloat16
        self.T = T
        self.w = torch.empty((T, k), dtype=f32, device=device)
        self.idx = torch.empty((T, k), dtype=i32, device=device)
        self.offsets = torch.empty((arch.num_experts + 1,), dtype=i32, device=device)
        self.perm = torch.empty((T * k,), dtype=i32, device=device)
        self.inv = torch.empty((T * k,), dtype=i32, device=device)
        self.h = torch.empty((T * k, arch.ffn), dtype=bf, device=device)
        self.y = torch.empty((T * k, H), dtype=f32, device=device)
        self.hd = torch.empty((T, max(arch.d_ffn, arch.shared_ffn)), dtype=bf, device=device)
        self.yd = torch.empty((T, H), dtype=f32, device=device)
        # tcgen05 path workspaces: gathered routed rows, split-K partials
        kmax = max(k, 1)
        self.xp = torch.empty((T * kmax, H), dtype=bf, device=device)
        from .kernels import tc_split, tc_units_workspace_floats, tc_workspace_floats

        need = 1
        for f in (arch.ffn, arch.d_ffn, arch.shared_ffn or arch.ffn):
            need = max(need, tc_workspace_floats(T * kmax, H, f, tc_split(H), tc_split(f)),
                       tc_units_workspace_floats(T * kmax, H, f))
        self.ysplit = torch.empty((need,), dtype=f32, device=device)
        self.pw = torch.empty((T, 64), dtype=f32, device=device)
        self.pidx = torch.empty((T, 64), dtype=i32, device=device)
        self.logits = torch.empty((T, arch.num_experts), dtype=f32, device=device)
        self._dense: dict[int, tuple[torch.Tensor, torch.Tensor]] = {}
        self.device = device

    def dense(self, T: int):
        """offsets {0, T} and identity permutation for a dense (1-expert) run."""
        if T not in self._dense:
            self._dense[T] = (
                torch.tensor([0, T], dtype=torch.int32, device=self.device),
                torch.arange(T, dtype=torch.int32, device=self.device),
            )
        return self._dense[T]


class SpecMoEEngine:
    def __init__(
        self,
        arch: ArchSpec,
        hw: HardwareSpec,
        timings: ProfiledTimings,
        policy: PolicySpec,
        *,
        batch: int = 1,
        seed: int | None = None,
        device=None,
        host_distinct: int | None = None,
        host_share: str | None = None,
        host_leader: bool = True,
        model_state: tuple | None = None,
        draft_perturb: float = 0.0,
        window_tokens: int = 1,
        max_tokens: int = 1024,
        record_timeline: bool = False,
        record: bool = False,
        record_routing: bool = False,
        capture_layers: tuple[int, ...] = (),
        cuda_graphs: bool = True,
        ffn_impl: str = "auto",
        tc_min_tokens: int | None = None,
        k3_units: bool = True,
        expert_parallel: bool = False,
        ep_group=None,
        host_codec: str | None = "auto",
        n_staging: int = 3,
    ):
        if ffn_impl not in ("auto", "tcgen05", "cuda_core"):
            raise ValueError("ffn_impl must be auto | tcgen05 | cuda_core")
        self.ffn_impl = ffn_impl
        # per-expert kernel rule (see _use_tc): tcgen05 at every token count.
        # A lone 1-2 token Mixtral expert streams faster on the CUDA-core
        # kernel (76 vs 83 us), but splitting a layer's late experts across
        # two kernel paths halves the launch sizes: one path keeps the SD
        # iteration time (851.6 vs 850.5 ms) and lifts in-situ K3 from 0.68
        # to 0.73 of the copy peak; small experts (DeepSeek /
        # Qwen) win on tcgen05 at any count (4.4 vs 2.9 TB/s)
        if tc_min_tokens is None:
            tc_min_tokens = 1
        self.tc_min_tokens = tc_min_tokens
        # verify-sized experts (<= 16 tokens) take the unit-fused tcgen05 K3
        # (one launch for both phases); False keeps the two-phase one
        self.k3_units = k3_units
        # test hook: treat every resident expert as late (one launch each), to
        # check that outputs do not depend on launch grouping
        self.force_late = False
        if not torch.cuda.is_available():
            raise RuntimeError("SpecMoEEngine needs a CUDA device (there is no CPU fallback)")
        self.num_sms = torch.cuda.get_device_properties(device if device is not None else 0).multi_processor_count
        self.arch = arch
        self.model = model_spec_for(arch)
        self.hw, self.timings, self.policy = hw, timings, policy
        self.batch = batch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.seed = policy.seed if seed is None else seed
        self.capacity = cache_capacity_slots(self.model, hw, policy)
        # expert parallelism (ep.py): this rank computes only its own block of
        # every layer's routed experts; its slot pool caches only those
        self.ep = None
        per_layer = arch.num_experts
        if expert_parallel:
            from .ep import ExpertParallelExchange

            if policy.policy not in (Policy.ON_DEMAND, Policy.DRAFT_PREFETCH):
                raise ValidationError("expert_parallel runs the on_demand or draft_prefetch policy")
            self.ep = ExpertParallelExchange(arch.num_experts, arch.top_k, ep_group)
            per_layer = len(self.ep.local_experts)
        if self.capacity < per_layer:
            raise ValidationError(
                f"cache capacity {self.capacity} is below experts_per_layer {per_layer}; "
                "a single layer could not be loaded"
            )
        self.capacity = min(self.capacity, arch.num_layers * per_layer)
        torch.cuda.set_device(self.device)
        if model_state is not None:
            # reuse another engine's pinned host pool and device weights
            # (sweeps over policy / batch / budget on one model)
            self.host_pool, self.weights = model_state
            self._owns_model = False
        else:
            if host_codec == "auto":
                # XC whenever the expert's matrices are whole coding blocks
                from .codec import codec_applies, expert_segments

                host_codec = "xc" if codec_applies(expert_segments(arch.ffn, arch.hidden)) else None
            self.host_pool = HostExpertPool(arch, host_distinct, share=host_share, leader=host_leader,
                                            codec=host_codec)
            self.weights = build_weights(arch, self.seed, self.device, self.host_pool, draft_perturb=draft_perturb)
            self._owns_model = True
        self.pool = torch.empty((self.capacity, arch.expert_elems), dtype=torch.bfloat16, device=self.device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.cache = NativeExpertCache(
            self.capacity,
            arch.num_layers,
            arch.num_experts,
            dev_pool_ptr=self.pool.data_ptr(),
            host_pool_ptr=self.host_pool.ptr,
            host_index=self.host_pool.index,
            slot_bytes=arch.expert_bytes,
            copy_stream_ptr=self.copy_stream.cuda_stream,
            batched_io=policy.batched_io,
        )
        self.staging = None
        self.decode_stream = None
        if self.host_pool.codec == "xc":
            # XC host tier: blobs land in staging buffers on the copy stream
            # and are expanded into their slots on the decode stream
            stride = self.host_pool.row_stride
            self.staging = torch.empty((n_staging * stride,), dtype=torch.uint8, device=self.device)
            self.decode_stream = torch.cuda.Stream(device=self.device)
            self.cache.set_codec(stride, self.staging.data_ptr(), stride, n_staging, self.decode_stream.cuda_stream)
        self.window_tokens = window_tokens
        self.cutoff_source = "explicit" if policy.cutoff_layer is not None else "solver"
        self.cutoff = (
            effective_cutoff(self.model, hw, timings, policy, window_tokens)
            if policy.policy is Policy.DRAFT_PREFETCH
            else None
        )
        if self.ep is not None:
            self.cutoff = self.ep.agree(self.cutoff)  # one predictor exchange schedule for all ranks
        N = policy.draft_length
        self.max_tokens = max_tokens
        self.draft_kv = KVCache(arch, batch, self.device, max_seq=min(arch.max_seq, max_tokens + N + 8))
        self.target_kv = KVCache(arch, batch, self.device, max_seq=min(arch.max_seq, max_tokens + N + 8))
        T_max = max(batch * (N + 1), batch * 2, 1)
        self.scratch = _Scratch(arch, T_max, self.device)
        self.prefill_scratch: _Scratch | None = None
        self.ep_scratch: _Scratch | None = None
        pk = policy.prefetch_k
        self.predictor = DraftGuidedPredictor(entries=max(N, 1) * arch.num_layers + 1, width=batch * pk)
        self.pred_w = torch.empty((batch, pk), dtype=torch.float32, device=self.device)
        self.pred_idx = torch.empty((batch, pk), dtype=torch.int32, device=self.device)
        # mapped host buffer receiving verify routing (zero-copy hand-off)
        self.route_ring = DraftGuidedPredictor(entries=1, width=max(T_max * arch.top_k, 1))
        self._lib = _native.load()
        _ev = C.c_void_p()
        _native.check("spmoe_event_create", self._lib.spmoe_event_create(C.byref(_ev)))
        self._route_ev = _ev.value
        self.use_graphs = cuda_graphs and not (
            policy.policy is Policy.DRAFT_PREFETCH and not policy.worker_prefetch
        )
        self._graphs_ready = False
        self.history = HistoryCounter(arch.num_layers, arch.num_experts)
        self._history_bufs: list[np.ndarray] = []
        self.use_worker = policy.worker_prefetch and policy.policy in (Policy.DRAFT_PREFETCH, Policy.COARSE_HISTORY)
        if self.use_worker:
            self.cache.start_worker()
        self.record_timeline = record_timeline
        self.record = record
        self.record_routing = record_routing
        self.trace_scores: list[list[np.ndarray]] = [[] for _ in range(batch)]
        self._iter_logits: list[torch.Tensor] = []
        self.capture_layers = set(capture_layers)
        self.time_k3 = False
        self.k3_events: list = []
        self._reset_run_state()

    # ------------------------------------------------------------------ utils
    def _reset_run_state(self) -> None:
        self.stalls: list[_Stall] = []
        self.iter_records: list[IterationRecord] = []
        self.slots: list[ComputeSlot] = []
        self._slot_events: list = []
        self.route_events: list = []  # (iteration, layer, event) with record_timeline
        self.iter_events: list[tuple[torch.cuda.Event, torch.cuda.Event, torch.cuda.Event]] = []
        self.draft_ms = 0.0
        self.verify_ms = 0.0
        self.stall_ms = {"prefetch": 0.0, "demand": 0.0}
        self.accepted_total = 0
        self.drafted_total = 0
        self.emitted_total = 0
        self._pending_gating: list[tuple[int, int]] = []  # (layer, slot) waits for gating_next_layer
        self._pushed: list[tuple[int, object]] = []  # (layer, ring row | host array) not yet logged
        # program-order log of cache-mutating decisions, for oracle replay:
        # ("task", layer, ids) when a prefetch task is consumed, ("verify",
        # layer, routed ids) at each verify layer
        self.decisions: list[tuple[str, int, list[int]]] = []
        self.captures: list[dict] = []
        # finished timing events folded into plain numbers (_fold_events), so
        # a long generate() holds a bounded number of live CUDA events
        self._stall_done = {"prefetch": 0.0, "demand": 0.0}
        self._prefetch_stall_by_layer: dict[int, float] = {}
        self._iters_done: list[tuple[float, float]] = []  # (draft ms, verify ms)
        self._k3_done: list[tuple[float, int, int, int]] = []  # (ms, bytes, experts, rows)
        self._k3_ev_ms: list[float] = []  # CUDA-event durations (time_k3 == "events")
        self.k3_events = []
        self._k3_spans = getattr(self, "_k3_spans", None)
        if self._k3_spans is not None:
            self._k3_spans.zero_()
        self._k3_span_next = 0
        self._slots_done: list[ComputeSlot] = []

    @property
    def stream(self):
        return torch.cuda.current_stream(self.device)

    def close(self) -> None:
        try:
            self.cache.stop_worker()
            torch.cuda.synchronize(self.device)
            self.cache.close()
        finally:
            self.predictor.close()
            self.route_ring.close()
            self._lib.spmoe_event_destroy(self._route_ev)
            if self._owns_model:
                self.host_pool.close()

    def _probe_cutoff(self, layer: int, steps: int) -> float | None:
        """Run `steps` SD iterations with drafting-stage prefetch up to
        `layer` and return the hidden fraction of `layer`'s prefetch copies
        (the measurement state is reset before and after)."""
        self.cutoff = layer
        if self._graphs_ready:
            torch.cuda.synchronize(self.device)
            self._graphs_ready = False
            self._ensure_graphs()
        self._reset_run_state()
        self.cache.clear_log()
        for _ in range(steps):
            self.step()
        torch.cuda.synchronize(self.device)
        hf = self.layer_hidden_fraction(layer)
        self._reset_run_state()
        self.cache.clear_log()
        return hf

    def recalibrate(self, timings: ProfiledTimings | None = None, probe_steps: int = 2) -> ProfiledTimings:
        """Replace the latency-model inputs with measurements of this engine
        (:func:`calibrate.measure_timings`), re-solve the cutoff layer and,
        if it moved, re-capture the draft-step graphs (they contain the
        predictor launches of layers <= cutoff).  When the solver finds even
        L = 0 infeasible, ``probe_steps`` iterations at L = 0 decide
        (``cutoff_source`` records which rule set the cutoff)."""
        from .calibrate import measure_timings

        t = timings if timings is not None else measure_timings(self)
        self.timings = t
        if self.policy.policy is Policy.DRAFT_PREFETCH:
            # distinct experts actually prefetched per prefetched layer per
            # iteration (each of the N draft tokens predicts its own top-k)
            n_it = max(1, len(self.iter_records))
            pre = sum(len(r.experts) for r in self.transfers() if r.kind is TransferKind.PREFETCH)
            layers = (self.cutoff + 1) if self.cutoff is not None else 0
            self.k_eff = max(self.policy.prefetch_k, round(pre / (n_it * layers))) if layers else None
            new = effective_cutoff(self.model, self.hw, t, self.policy, self.window_tokens, self.k_eff)
            self.cutoff_source = "explicit" if self.policy.cutoff_layer is not None else "solver"
            if (new is None and self.policy.cutoff_layer is None and self.cutoff is not None and probe_steps > 0
                    and self.seqs):
                # the analytic window test failed even at L = 0 (k_eff copies
                # do not fit in the measured drafting window).  Measure
                # instead: run `probe_steps` iterations at L = 0 and keep it
                # if the verify waited on those prefetches for less than 0.2
                # of their copy time (the paper's >= 0.8 hidden target),
                # rather than degenerating to on-demand with the link idle
                # through the whole drafting stage.
                hf = self._probe_cutoff(0, probe_steps)
                if hf is not None and hf >= 0.8:
                    new = 0
                    self.cutoff_source = f"measured (solver infeasible; L=0 prefetch copies {hf:.2f} hidden)"
            if self.ep is not None:
                new = self.ep.agree(new)
            if new != self.cutoff:
                self.cutoff = new
                if self._graphs_ready:
                    torch.cuda.synchronize(self.device)
                    self._graphs_ready = False
                    self._ensure_graphs()
        return t

    def layer_hidden_fraction(self, layer: int) -> float | None:
        """1 - (verify stalls on layer `layer`'s in-flight prefetches) /
        (that layer's prefetch copy time), over the recorded run; None
        without prefetches there."""
        self._fold_events(force=True)
        pre = sum(t.duration for t in self.transfers() if t.kind is TransferKind.PREFETCH and t.layer == layer) * 1e3
        if pre <= 0:
            return None
        return 1.0 - self._prefetch_stall_by_layer.get(layer, 0.0) / pre

    @property
    def wire_ratio(self) -> float:
        """Host-link bytes per raw expert byte (1.0 on the raw tier)."""
        hp = self.host_pool
        return (sum(hp.wire) / len(hp.wire)) / self.arch.expert_bytes if hp.codec else 1.0

    def effective_hw(self) -> HardwareSpec:
        """``hw`` with pcie_bandwidth in RAW expert bytes per second: the link
        peak divided by the wire ratio, so the reference's floor
        t_io >= expert_size / pcie_bandwidth (config.py:362-375) and the
        cutoff model's I/O term describe the XC tier correctly."""
        from dataclasses import replace

        return replace(self.hw, pcie_bandwidth=self.hw.pcie_bandwidth / self.wire_ratio)

    @property
    def model_state(self) -> tuple:
        """(host pool, device weights) to share with another engine."""
        return self.host_pool, self.weights

    # ------------------------------------------------------------- MoE layers
    def _drain(self) -> None:
        """Wait for the worker to consume every pushed task; log them in FIFO
        (= consumption) order."""
        self.cache.drain()
        if self.record:
            for layer, src in self._pushed:
                ids = [int(v) for v in (self.predictor.view[src] if isinstance(src, int) else src)]
                self.decisions.append(("task", layer, ids))
        self._pushed = []

    def _k3_path(self, F: int, ntok: int) -> str:
        """Kernel for ONE expert with ``ntok`` routed tokens: "cc" (the
        CUDA-core, bit-exact path: ``ffn_impl="cuda_core"`` or fewer than
        ``tc_min_tokens`` tokens), "units" (the unit-fused tcgen05 kernel,
        <= 16 tokens: the verify regime) or "tc" (the two-phase tcgen05
        kernels, more tokens: prefill, large batches).  Decided per expert,
        never per launch, so an expert's output bits do not depend on which
        experts happen to share its launch (that depends on copy timing)."""
        if self.ffn_impl == "cuda_core" or self.arch.hidden % 128 or F % 128:
            return "cc"
        if self.ffn_impl != "tcgen05" and ntok < self.tc_min_tokens:
            return "cc"
        return "units" if (self.k3_units and ntok <= K.UNIT_MAX_TOKENS) else "tc"

    def _use_tc(self, F: int, ntok: int) -> bool:
        return self._k3_path(F, ntok) != "cc"

    def _ffn(self, pool, slots, mask, xn, F, k, offsets, perm, h, y, maxtok, s: _Scratch, counts=None,
             use_tc=None) -> None:
        """K3 for the experts in ``mask``, all on one path (``use_tc``: a
        :meth:`_k3_path` name, or by default the path of ``maxtok`` tokens);
        ``counts`` = routed tokens of each of those experts (host-known)."""
        path = use_tc if isinstance(use_tc, str) else self._k3_path(F, maxtok)
        rows = xn.shape[0] * k
        if path == "units":
            K.expert_ffn_tc_units(pool, slots, mask, xn, F, k, offsets, perm, maxtok, None, None, y, s.ysplit)
        elif path == "tc":
            # launch-independent split: bits do not depend on launch grouping
            su, sd = K.tc_plan_static(self.arch.hidden, F, self.num_sms)
            K.expert_ffn_tc(pool, slots, mask, xn, F, k, offsets, perm, s.xp[:rows], h, y, s.ysplit, su, sd)
        else:
            K.expert_ffn(pool, slots, mask, xn, F, k, offsets, perm, h, y, maxtok)

    def _dense_ffn(self, blob: torch.Tensor, F: int, xn: torch.Tensor, resid: torch.Tensor, s: _Scratch, out=None):
        T = xn.shape[0]
        off, perm = s.dense(T)
        self._ffn(blob, [0], 1, xn, F, 1, off, perm, s.hd, s.yd, T, s)
        return K.moe_combine(s.yd, perm, None, T, self.arch.hidden, 1, residual=resid, out=out)

    def _draft_ffn(self, l: int, xn: torch.Tensor, resid: torch.Tensor, s: _Scratch) -> torch.Tensor:
        """The draft's MLP at layer l: its dense FFN; with a sigmoid-gated
        shared expert (Qwen1.5-MoE) the mean-expert FFN plus the target's
        shared expert under its per-token gate (K1's shared-gate output),
        combined by K4 like the target's shared path."""
        a, lw = self.arch, self.weights.layers[l]
        if not (a.shared_gate and lw.shared is not None and lw.shared_gate is not None):
            return self._dense_ffn(lw.draft_ffn, a.d_ffn, xn, resid, s)
        T = xn.shape[0]
        off, pm = s.dense(T)
        self._ffn(lw.draft_ffn, [0], 1, xn, a.d_ffn, 1, off, pm, s.hd, s.yd, T, s)
        ys = s.y[:T]
        self._ffn(lw.shared, [0], 1, xn, a.shared_ffn, 1, off, pm, s.hd, ys, T, s)
        _, _, _, sg = K.router_topk(xn, lw.router, 1, a.renorm, shared_gate_w=lw.shared_gate)
        return K.moe_combine(s.yd, pm, None, T, a.hidden, 1, residual=resid, y_shared=ys, shared_gate=sg)

    def _timed_ffn(self, experts, counts, slots, mask, xn, offsets, perm, s, maxtok, k=None) -> None:
        """K3 over ``experts`` (one launch per kernel path: experts are
        grouped by their own token counts); with ``time_k3`` set, brackets
        each launch with CUDA events and books its algorithmic bytes (weights
        of every expert in the mask read once + activations in/out) for the
        roofline."""
        a = self.arch
        k = a.top_k if k is None else k
        groups: dict[str, list[int]] = {}
        for e in experts:
            groups.setdefault(self._k3_path(a.ffn, int(counts[e])), []).append(e)
        for path, grp in groups.items():
            self._timed_ffn_group(grp, counts, slots, sum(1 << e for e in grp), xn, offsets, perm, s, k, path)

    def _timed_ffn_group(self, experts, counts, slots, mask, xn, offsets, perm, s, k, use_tc) -> None:
        a = self.arch
        cnt = [int(counts[e]) for e in experts]
        maxtok = max(cnt) if cnt else 0
        if not self.time_k3:
            self._ffn(self.pool, slots, mask, xn, a.ffn, k, offsets, perm, s.h, s.y, maxtok, s, cnt, use_tc)
            return
        # device-clock span of the call (first kernel's first CTA start ->
        # last kernel's last CTA end): CUDA events around launches are skewed
        # by tens of microseconds while the host link is saturated
        # (profiles/r2_event_skew_probe.txt); time_k3 == "events" also
        # brackets the call with CUDA events for comparison
        if self._k3_spans is None:
            self._k3_spans = torch.zeros((1 << 16, 2), dtype=torch.int64, device=self.device)
        slot = self._k3_span_next % self._k3_spans.shape[0]
        self._k3_span_next += 1
        self._lib.spmoe_k3_devtiming(self._k3_spans[slot].data_ptr())
        ea = eb = None
        if self.time_k3 == "events":
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()  # creates the events; the launcher re-records them
            eb.record()
            # the C launcher records ea right before its first kernel and eb
            # after its last, so host-side launch preparation is not counted
            self._lib.spmoe_k3_timing(ea.cuda_event, eb.cuda_event)
        self._ffn(self.pool, slots, mask, xn, a.ffn, k, offsets, perm, s.h, s.y, maxtok, s, cnt, use_tc)
        self._lib.spmoe_k3_devtiming(None)
        rows = int(sum(int(counts[e]) for e in experts))
        act = rows * (a.hidden * 2 + 2 * a.ffn * 2 + a.hidden * 4)  # x in, h out+in, y out
        self.k3_events.append((ea, eb, len(experts) * a.expert_bytes + act, len(experts), rows, slot))

    def k3_roofline(self) -> dict:
        """Average algorithmic bytes / launch-pair duration of the timed K3 calls."""
        self._fold_events(force=True)
        done = self._k3_done
        if not done:
            return {}
        ms = [x[0] for x in done]
        byts = [x[1] for x in done]
        tot_ms = sum(ms)
        return {
            "launches": len(ms),
            "bytes_per_launch": sum(byts) / len(byts),
            "ms_per_launch": tot_ms / len(ms),
            "achieved_gbs": sum(byts) / (tot_ms / 1e3) / 1e9,
            "experts_per_launch": sum(x[2] for x in done) / len(ms),
            "rows_per_launch": sum(x[3] for x in done) / len(ms),
            "total_ms": tot_ms,
            "by_shape": self._k3_by_shape(done),
            "clock": "device globaltimer span per call (first CTA start -> last CTA end)",
            "events_ms_per_launch": (sum(self._k3_ev_ms) / len(self._k3_ev_ms)) if self._k3_ev_ms else None,
        }

    def _k3_by_shape(self, done) -> dict:
        """Timed K3 launches grouped by (experts, routed rows): count, mean
        microseconds and achieved GB/s of algorithmic bytes."""
        groups: dict = {}
        for t, byts, ne, rows in done:
            g = groups.setdefault(f"{ne}x{rows}", [0, 0.0, 0])
            g[0] += 1
            g[1] += t
            g[2] += byts
        return {k: {"n": v[0], "us": round(v[1] / v[0] * 1e3, 1), "gbs": round(v[2] / (v[1] / 1e3) / 1e9, 1)}
                for k, v in sorted(groups.items(), key=lambda kv: -kv[1][0])}

    def _route(self, l: int, xn: torch.Tensor, s: _Scratch):
        """K1 on the verify tokens; indices also land in the mapped route ring
        (zero-copy hand-off to the host), then the route event is recorded
        (as an external graph node when captured)."""
        a = self.arch
        lw = self.weights.layers[l]
        T = xn.shape[0]
        w, idx, _, sg = K.router_topk(
            xn,
            lw.router,
            a.top_k,
            a.renorm,
            host_idx_dev_ptr=self.route_ring.dev_ptr,
            shared_gate_w=lw.shared_gate,
            out=(s.w[:T], s.idx[:T]),
            logits_out=s.logits[:T] if self.record_routing else None,
        )
        self._lib.spmoe_event_record_external(self._route_ev, self.stream.cuda_stream)
        return w, idx, sg

    def _moe_verify(self, l: int, xn: torch.Tensor, resid: torch.Tensor, s: _Scratch, routed=None) -> torch.Tensor:
        a = self.arch
        lw = self.weights.layers[l]
        T, H = xn.shape
        k, E = a.top_k, a.num_experts
        w, idx, sg = routed if routed is not None else self._route(l, xn, s)
        gating = self.policy.policy is Policy.GATING_NEXT_LAYER and l + 1 < a.num_layers
        if gating:
            # K1 for layer l+1 runs on the GPU now; its task is pushed after
            # layer l's lookups and demand load (simcore.py:360-418 order)
            g_ring = self._gating_launch(l + 1, xn)
        self._lib.spmoe_event_synchronize(self._route_ev)
        ids = self.route_ring.view[0, : T * k].copy()
        counts = np.bincount(ids, minlength=E)
        # copies first: the host-side bookkeeping below overlaps the link
        plan = self._cache_issue(l, counts) if self.ep is None else None
        if self.record:
            self.decisions.append(("verify", l, [int(v) for v in ids]))
        if gating:
            self._gating_push(l + 1, g_ring)
        self.history.record_many(l, ids)
        if self.record_routing:
            self._iter_logits.append(s.logits[:T].clone())
        if self.ep is not None:
            return self._moe_verify_ep(l, xn, resid, s, w, idx, sg, ids)
        offsets, perm, inv = K.moe_permute(idx, E, out=(s.offsets, s.perm[: T * k], s.inv[: T * k]))
        slots = self._run_plan(l, plan, counts, xn, k, offsets, perm, s)
        return self._shared_and_combine(l, xn, resid, s, w, idx, sg, s.y, inv, slots)

    def _run_experts(self, l: int, counts: np.ndarray, x: torch.Tensor, k: int, offsets, perm, s: _Scratch) -> list:
        """Cache decisions + K3 for the experts with ``counts > 0`` at layer l:
        touch the union in ascending order, demand-load the misses behind
        queued prefetches, run the resident experts first and the late ones
        after their slots' ready events (§4.3; all late experts but
        the last in one launch under the last one's copy, then the last),
        then record the slots' read events.  Returns the slot of every expert (0 if unused)."""
        return self._run_plan(l, self._cache_issue(l, counts), counts, x, k, offsets, perm, s)

    def _cache_issue(self, l: int, counts: np.ndarray) -> tuple:
        """The layer's cache decisions, in the reference order: touch the
        required experts ascending (lookup, cache.py:62-77), then demand-load
        the misses as one batch behind queued prefetches (on_demand_load,
        prefetch.py:276-301) -- issued before any other host work of the
        layer so the link starts as soon as routing is known."""
        required = [int(e) for e in np.nonzero(counts)[0]]
        hits, missing = [], []
        for e in required:
            (hits if self.cache.lookup(ExpertId(l, e), touch=True) else missing).append(e)
        slot = {}
        if missing:
            for e, sl in zip(missing, self.cache.demand_load([ExpertId(l, e) for e in missing])):
                slot[e] = sl
        ready, late_prefetch = [], []
        for e in hits:
            slot[e] = self.cache.slot_of(l, e)
            (ready if self.cache.slot_ready(slot[e]) and not self.force_late else late_prefetch).append(e)
        return required, slot, ready, late_prefetch, missing

    def _run_plan(self, l: int, plan: tuple, counts: np.ndarray, x: torch.Tensor, k: int, offsets, perm,
                  s: _Scratch) -> list:
        required, slot, ready, late_prefetch, missing = plan
        E = self.arch.num_experts
        stream_ptr = self.stream.cuda_stream
        slots = [slot.get(e, 0) for e in range(E)]
        maxtok = int(counts.max()) if counts.size else 0
        if ready:
            mask = sum(1 << e for e in ready)
            self._timed_ffn(ready, counts, slots, mask, x, offsets, perm, s, maxtok, k)
        # late experts land one by one (prefetches in flight first, then the
        # demand batch in copy order); the layer cannot end before the LAST
        # one lands, so every earlier late expert runs in ONE launch once the
        # second-to-last has landed (under the last one's copy), and only the
        # last expert's K3 stays on the critical path.  Same layer latency as
        # running each expert on arrival, far fewer single-expert launches.
        late = [("prefetch", e) for e in late_prefetch] + [("demand", e) for e in missing]
        for batch in ([late[:-1], late[-1:]] if len(late) > 1 else [late]):
            if not batch:
                continue
            for kind, e in batch:
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ea.record()
                self.cache.wait_slot(slot[e], stream_ptr)
                eb.record()
                self.stalls.append(_Stall(kind, l, ea, eb))
            grp = [e for _, e in batch]
            self._timed_ffn(grp, counts, slots, sum(1 << e for e in grp), x, offsets, perm, s,
                            max(int(counts[e]) for e in grp), k)
        for e in required:
            self.cache.mark_read(slot[e], stream_ptr)
        return slots

    def _shared_and_combine(self, l, xn, resid, s, w, idx, sg, y, inv, slots):
        a = self.arch
        lw = self.weights.layers[l]
        T, H = xn.shape
        ys = None
        if lw.shared is not None:
            off, pm = s.dense(T)
            self._ffn(lw.shared, [0], 1, xn, a.shared_ffn, 1, off, pm, s.hd, s.yd, T, s)
            ys = s.yd
        if l in self.capture_layers:
            cap = {"layer": l, "xn": xn.clone(), "resid": resid.clone(), "idx": idx.clone(), "w": w.clone(),
                   "slots": list(slots), "sg": None if sg is None else sg.clone()}
        out = K.moe_combine(y, inv, w, T, H, a.top_k, residual=resid, y_shared=ys, shared_gate=sg, out=resid)
        if l in self.capture_layers:
            cap["out"] = out.clone()
            self.captures.append(cap)
        return out

    def _moe_verify_ep(self, l, xn, resid, s, w, idx, sg, ids) -> torch.Tensor:
        """Expert-parallel verify MoE (ep.py): dispatch routed rows to the
        experts' owners, run this rank's experts on what it received, send the
        outputs back, combine.  Every rank must call this for every layer."""
        a = self.arch
        T, H = xn.shape
        k, E = a.top_k, a.num_experts
        offsets, perm, inv = K.moe_permute(idx, E, out=(s.offsets, s.perm[: T * k], s.inv[: T * k]))
        counts = np.bincount(ids, minlength=E)
        x_recv, e_recv, e_host = self.ep.dispatch(xn, perm, counts)
        R = x_recv.shape[0]
        slots = [0] * E
        if R:
            if self.ep_scratch is None or self.ep_scratch.T < R:
                self.ep_scratch = _Scratch(a, max(R, self.ep.world * self.scratch.T), self.device)
            es = self.ep_scratch
            off2, perm2, inv2 = K.moe_permute(e_recv.view(R, 1), E, out=(es.offsets, es.perm[:R], es.inv[:R]))
            slots = self._run_experts(l, np.bincount(e_host, minlength=E), x_recv, 1, off2, perm2, es)
            y_recv = K.gather_rows(es.y, inv2, 1)
        else:
            y_recv = torch.empty((0, H), dtype=torch.float32, device=self.device)
        y_back = self.ep.combine(y_recv)
        return self._shared_and_combine(l, xn, resid, s, w, idx, sg, y_back, inv, slots)

    def _gating_launch(self, layer: int, xn: torch.Tensor) -> tuple:
        """gating_next_layer baseline, GPU half: K1 predicts layer+1 from this
        layer's MLP input (one token per sequence: the verify position, as
        simcore.py:407 uses ``position`` -- the first of each sequence's
        verify tokens)."""
        pk = self.policy.prefetch_k
        B = self.batch
        x_pos = xn.view(B, -1, xn.shape[-1])[:, 0, :].contiguous()
        return self.predictor.predict(
            x_pos, self.weights.layers[layer].router, pk, True, self.scratch.pw[:B, :pk], self.scratch.pidx[:B, :pk]
        )

    def _gating_push(self, layer: int, launched: tuple) -> None:
        """gating_next_layer baseline, host half: blocking prefetch of the
        predicted layer+1 experts (``vanilla_prefetch_step``,
        prefetch.py:241-273), issued after this layer's demand load."""
        pk = self.policy.prefetch_k
        B = self.batch
        i, hptr, ev = launched
        self.cache.push_task(layer, hptr, B * pk, ev)
        self._pushed.append((layer, i))
        self._drain()
        for e in set(int(v) for v in self.predictor.view[i][: B * pk] if v >= 0):
            sl = self.cache.slot_of(layer, e)
            if sl >= 0:
                self._pending_gating.append((layer, sl))

    # -------------------------------------------------------------- forwards
    def _embed(self, tokens: torch.Tensor) -> torch.Tensor:
        return self.weights.embed[tokens]

    def _draft_forward(self, tokens: torch.Tensor, start: torch.Tensor, kv_len_max: int, predict_step: int | None,
                       ring_base: int | None = None):
        """Draft pass over ``tokens`` [B, T]; returns last-token logits [B, V] f32.
        ``predict_step`` (iteration-local draft step index) enables Algorithm 1
        at layers <= cutoff: eagerly (predict + push per layer) or, with
        ``ring_base`` set (CUDA-graph capture), K1 into ring entry
        ring_base + l plus an external event node; the host pushes the tasks
        after launching the graph."""
        a, w = self.arch, self.weights
        B, T = tokens.shape
        x = self._embed(tokens)
        s = self.scratch if B * T <= self.scratch.T else self._prefill_scratch(B * T)
        spmoe = predict_step is not None and self.cutoff is not None
        pk = self.policy.prefetch_k
        for l in range(a.num_layers):
            lw = w.layers[l]
            x = attention_block(w, l, x, self.draft_kv, start)
            hn = rms_norm(x, lw.ffn_norm, a.rms_eps)
            if spmoe and l <= self.cutoff:
                if ring_base is None:
                    self._predict_and_enqueue(l, hn[:, -1, :].contiguous(), predict_step)
                else:
                    self.predictor.predict_at(ring_base + l, hn[:, -1, :].contiguous(), lw.router, pk, True,
                                              self.pred_w, self.pred_idx)
            x = self._draft_ffn(l, hn.reshape(B * T, -1), x.reshape(B * T, -1), s).view(B, T, -1)
        return lm_logits(w, x[:, -1, :])

    # ------------------------------------------------------------ CUDA graphs
    def _capture(self, fn) -> torch.cuda.CUDAGraph:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            fn()  # warm-up outside capture (kernel selection, workspaces)
        torch.cuda.current_stream(self.device).wait_stream(side)
        # thread_local: the prefetch worker thread may call CUDA (event
        # queries, copies on its own stream) while the main thread captures.
        # Python's GC stays off during the capture: a collected object whose
        # finaliser frees pinned or device memory (cudaFreeHost, cudaFree) on
        # this thread would invalidate it (seen when earlier work in the
        # process left such objects in reference cycles)
        import gc

        gc_on = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                fn()
        finally:
            if gc_on:
                gc.enable()
        return g

    def _ensure_graphs(self) -> None:
        """Capture, once per engine (after prefill): one graph per draft step
        (embed, 32 layers with attention, predictor K1 + external event
        nodes, dense FFN, lm_head, argmax) and one graph per verify layer for
        the pre-MoE block (norm, attention, norm, router K1 + route event).
        Static buffers: base positions, step-0 tokens, draft tokens, the
        verify residual stream and MLP input."""
        if self._graphs_ready or not self.use_graphs:
            return
        a, B, N = self.arch, self.batch, self.policy.draft_length
        dev = self.device
        L, H = a.num_layers, a.hidden
        T = N + 1
        self._g_base = torch.zeros((B,), dtype=torch.int64, device=dev)
        self._g_tok0 = torch.zeros((B, 2), dtype=torch.int64, device=dev)
        self._g_draft = torch.zeros((B, N), dtype=torch.int32, device=dev)
        self._h_base = torch.zeros((B,), dtype=torch.int64).pin_memory()
        self._h_tok0 = torch.zeros((B, 2), dtype=torch.int64).pin_memory()
        self._vx = torch.zeros((B * T, H), dtype=torch.bfloat16, device=dev)
        self._vxn = torch.zeros((B * T, H), dtype=torch.bfloat16, device=dev)
        self._vstart = torch.zeros((B,), dtype=torch.int64, device=dev)
        self._h_vstart = torch.zeros((B,), dtype=torch.int64).pin_memory()
        # each sequence's own next positions for the warm-up run outside
        # capture: it writes KV only at positions the next real step rewrites
        # before reading them (draft P-2.., verify P-1..), never over
        # committed entries of a longer sequence (re-capture mid-run with
        # diverged lengths, see recalibrate)
        for b, sq in enumerate(self.seqs):
            self._h_base[b] = len(sq) - 2
            self._h_vstart[b] = len(sq) - 1
        self._g_base.copy_(self._h_base)
        self._vstart.copy_(self._h_vstart)
        dkv, tkv = self.draft_kv.max_seq, self.target_kv.max_seq

        def draft_fn(d):
            def fn():
                if d == 0:
                    tok, start = self._g_tok0, self._g_base
                else:
                    tok, start = self._g_draft[:, d - 1 : d].long(), self._g_base + (d + 1)
                logits = self._draft_forward(tok, start, dkv, d, ring_base=d * L)
                self._g_draft[:, d].copy_(K.argmax_rows(logits))
            return fn

        self._vroute: list = [None] * L

        def verify_fn(l):
            def fn():
                lw = self.weights.layers[l]
                x = self._vx.view(B, T, H)
                attention_block(self.weights, l, x, self.target_kv, self._vstart, out=x)
                rms_norm(x, lw.ffn_norm, a.rms_eps, out=self._vxn.view(B, T, H))
                self._vroute[l] = self._route(l, self._vxn, self.scratch)
            return fn

        self._draft_graphs = [self._capture(draft_fn(d)) for d in range(N)]
        self._verify_graphs = [self._capture(verify_fn(l)) for l in range(L)]
        torch.cuda.synchronize(dev)
        self._graphs_ready = True

    def _predict_and_enqueue(self, l: int, x_last: torch.Tensor, step: int) -> None:
        pk = self.policy.prefetch_k
        i, hptr, ev = self.predictor.predict(x_last, self.weights.layers[l].router, pk, True, self.pred_w, self.pred_idx)
        if self.ep is not None:
            self._ep_enqueue(l, i, step)
        else:
            self.cache.push_task(l, hptr, self.predictor.width, ev, step)
            self._pushed.append((l, i))
        if not self.policy.worker_prefetch:
            # vanilla executor: block until the copies are issued, and make the
            # next layer wait for them (prefetch.py:241-273)
            self._drain()
            sp = self.stream.cuda_stream
            for e in sorted(set(int(v) for v in self.predictor.view[i] if v >= 0)):
                sl = self.cache.slot_of(l, e)
                if sl >= 0 and not self.cache.slot_ready(sl):
                    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ea.record()
                    self.cache.wait_slot(sl, sp)
                    eb.record()
                    self.stalls.append(_Stall("prefetch", l, ea, eb))

    def _ep_enqueue(self, l: int, i: int, step: int) -> None:
        """Expert-parallel Algorithm 1 l.8-9 (ep.py): once predictor entry i
        has landed, every rank's predicted experts for layer l are gathered
        on the host and this rank enqueues the ones it owns (its cache is
        the one the verify reads).  The task's index array is host memory
        kept alive (in ``_pushed``) until the drain that logs it."""
        from . import _native

        _native.check("spmoe_event_synchronize", self._lib.spmoe_event_synchronize(self.predictor.events[i]))
        share = self.ep.prefetch_share(self.predictor.view[i].copy())
        if share.size:
            self.cache.push_task(l, share.ctypes.data, int(share.size), 0, step)
            self._pushed.append((l, share))

    def _target_forward(self, tokens: torch.Tensor, start: torch.Tensor, kv_len_max: int, s: _Scratch,
                        logits: bool = True) -> torch.Tensor | None:
        a, w = self.arch, self.weights
        B, T = tokens.shape
        x = self._embed(tokens)
        for l in range(a.num_layers):
            self._gating_waits(l)
            lw = w.layers[l]
            x = attention_block(w, l, x, self.target_kv, start)
            hn = rms_norm(x, lw.ffn_norm, a.rms_eps)
            x = self._moe_verify(l, hn.reshape(B * T, -1).contiguous(), x.reshape(B * T, -1).contiguous(), s).view(B, T, -1)
        return lm_logits(w, x) if logits else None

    def _step_graphed(self, P: list[int], N: int, ev1):
        """Drafting + verification with the captured graphs; the per-layer
        verify MoE (host cache logic, demand loads, K2-K4) stays eager."""
        a, B = self.arch, self.batch
        L, H, T = a.num_layers, a.hidden, N + 1
        for b, sq in enumerate(self.seqs):
            self._h_base[b] = P[b] - 2
            self._h_tok0[b, 0] = sq[-2]
            self._h_tok0[b, 1] = sq[-1]
            self._h_vstart[b] = P[b] - 1
        self._g_base.copy_(self._h_base, non_blocking=True)
        self._g_tok0.copy_(self._h_tok0, non_blocking=True)
        self._vstart.copy_(self._h_vstart, non_blocking=True)
        spmoe = self.cutoff is not None and self.policy.policy is Policy.DRAFT_PREFETCH
        width = self.predictor.width
        for d in range(N):
            self._slot_begin()
            self._draft_graphs[d].replay()
            self._slot_end("draft", P[0] - 1 + d, -1)
            if spmoe:
                # tasks are pushed after the graph is enqueued, so the worker
                # waits on this replay's event nodes (Algorithm 1 l.8-9)
                for l in range(self.cutoff + 1):
                    i = d * L + l
                    if self.ep is not None:
                        self._ep_enqueue(l, i, d)
                        continue
                    self.cache.push_task(l, self.predictor.host_ptr_of(i), width, self.predictor.events[i], d)
                    self._pushed.append((l, i))
        ev1.record(self.stream)
        if self.use_worker:
            self._drain()
        draft_tok = self._g_draft
        # verify: embed [last committed, drafts] into the static residual stream
        vtok = torch.cat([self._g_tok0[:, 1:2], draft_tok.long()], dim=1)
        self._vx.copy_(self._embed(vtok).view(B * T, H))
        for l in range(L):
            self._slot_begin()
            self._gating_waits(l)
            self._verify_graphs[l].replay()
            if self.record_timeline:
                # end of the layer's pre-MoE block (routing known on the GPU)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(self.stream)
                self.route_events.append((len(self.iter_records), l, ev))
            self._moe_verify(l, self._vxn, self._vx, self.scratch, routed=self._vroute[l])
            self._slot_end("verify", P[0] - 1, l)
        logits = lm_logits(self.weights, self._vx.view(B, T, H))
        return logits, draft_tok

    def _slot_begin(self) -> None:
        if self.record_timeline:
            self._slot_ev = torch.cuda.Event(enable_timing=True)
            self._slot_ev.record(self.stream)

    def _slot_end(self, kind: str, token: int, layer: int) -> None:
        """ComputeSlot timeline (simcore.py:69-76): one slot per draft step
        (layer -1 = the whole captured step) and per verify layer."""
        if self.record_timeline:
            e = torch.cuda.Event(enable_timing=True)
            e.record(self.stream)
            self._slot_events.append((kind, len(self.iter_records), token, layer, self._slot_ev, e))

    def _gating_waits(self, l: int) -> None:
        if not self._pending_gating:
            return
        sp = self.stream.cuda_stream
        waits = [sl for (ly, sl) in self._pending_gating if ly == l]
        self._pending_gating = [(ly, sl) for (ly, sl) in self._pending_gating if ly != l]
        for sl in waits:
            if not self.cache.slot_ready(sl):
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ea.record()
                self.cache.wait_slot(sl, sp)
                eb.record()
                self.stalls.append(_Stall("prefetch", l, ea, eb))

    def _prefill_scratch(self, T: int) -> _Scratch:
        if self.prefill_scratch is None or self.prefill_scratch.T < T:
            self.prefill_scratch = _Scratch(self.arch, T, self.device)
            if self.route_ring.width < T * self.arch.top_k:
                self.route_ring.close()
                self.route_ring = DraftGuidedPredictor(entries=1, width=T * self.arch.top_k)
        return self.prefill_scratch

    # ------------------------------------------------------------- SD loop
    def prefill(self, prompts: torch.Tensor) -> None:
        """Fill both KV caches with ``prompts[:, :-1]`` (not timed); the last
        prompt token is processed by the first draft step and verify."""
        B, P = prompts.shape
        if B != self.batch or P < 2:
            raise ValueError("prompts must be [batch, >=2]")
        self._check_room(P)
        self.seqs = [list(map(int, row)) for row in prompts.tolist()]
        self.draft_len = [P - 1] * B  # positions held by the draft KV
        ctx = prompts[:, :-1].to(self.device)
        start = torch.zeros((B,), dtype=torch.int64, device=self.device)
        s = self._prefill_scratch(B * (P - 1))
        self._draft_forward(ctx, start, P - 1, None)
        self._target_forward(ctx, start, P - 1, s, logits=False)
        self.cache.drain()
        torch.cuda.synchronize(self.device)
        self._ensure_graphs()
        self.cache.reset_stats()
        self.cache.clear_log()
        self.history = HistoryCounter(self.arch.num_layers, self.arch.num_experts)
        self._reset_run_state()

    def _check_room(self, positions: int) -> None:
        """Raise before any KV write past the caches: an SD iteration writes
        positions up to len(seq) + N - 1 (verify), prefill up to P - 2."""
        cap = min(self.draft_kv.max_seq, self.target_kv.max_seq)
        if positions > cap:
            raise ValueError(
                f"sequence would need {positions} KV positions but the caches hold {cap} "
                f"(max_tokens={self.max_tokens}, arch.max_seq={self.arch.max_seq})")

    def _coarse_history_enqueue(self) -> None:
        pk = self.policy.prefetch_k
        self._history_bufs = []
        for l in range(self.arch.num_layers):
            buf = np.array(top_k_indices(self.history.scores(l), pk), dtype=np.int32)
            self._history_bufs.append(buf)
            self.cache.push_task(l, buf.ctypes.data, pk, 0)
            self._pushed.append((l, buf))

    _LIVE_EVENTS = 2048

    def _fold_events(self, force: bool = False) -> None:
        """Turn completed timing-event pairs into numbers and drop the events
        once more than _LIVE_EVENTS are held (or always with ``force``).  The
        lists are appended in stream order and step() ends with a host sync,
        so everything recorded by earlier iterations has completed."""
        n = len(self.stalls) + len(self.k3_events) + len(self.iter_events) + len(self._slot_events)
        if not force and n <= self._LIVE_EVENTS:
            return
        torch.cuda.synchronize(self.device)
        for s_ in self.stalls:
            ms = s_.a.elapsed_time(s_.b)
            self._stall_done[s_.kind] += ms
            if s_.kind == "prefetch":
                self._prefetch_stall_by_layer[s_.layer] = self._prefetch_stall_by_layer.get(s_.layer, 0.0) + ms
        self.stalls = []
        if self.k3_events:
            n = min(self._k3_span_next, self._k3_spans.shape[0])
            spans = self._k3_spans[:n].cpu().numpy()
            self._k3_spans[:n].zero_()
            for ea, eb, byts, ne, rows, slot in self.k3_events:
                t0, t1 = int(spans[slot, 0]), int(spans[slot, 1])
                if ea is not None:
                    self._k3_ev_ms.append(ea.elapsed_time(eb))
                if t0 > 0 and t1 >= t0:
                    self._k3_done.append(((t1 - t0) / 1e6, byts, ne, rows))
                elif ea is not None:  # a path without device spans (CUDA-core K3)
                    self._k3_done.append((ea.elapsed_time(eb), byts, ne, rows))
            self._k3_span_next = 0
        self.k3_events = []
        for e0, e1, e2 in self.iter_events:
            self._iters_done.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
        self.iter_events = []
        for kind, it, tok, layer, ea, eb in self._slot_events:
            self._slots_done.append(ComputeSlot(kind, it, tok, layer, self.cache.since_epoch_ms(ea) / 1e3,
                                                self.cache.since_epoch_ms(eb) / 1e3))
        self._slot_events = []

    def step(self, remaining: list[int] | None = None) -> list[int]:
        """One SD iteration for every sequence; returns tokens emitted per
        sequence (the accepted drafts plus one correction/bonus token)."""
        self._fold_events()
        a, pol = self.arch, self.policy
        B = self.batch
        N = pol.draft_length
        if remaining is not None and B == 1 and self.ep is None:
            # (expert-parallel ranks draft in lockstep: they always draft N
            # and clip the emitted tokens below)
            N = max(1, min(N, remaining[0]))
        dev = self.device
        st = self.stream
        ev0, ev1, ev2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        self.predictor.reset()
        ev0.record(st)
        if pol.policy is Policy.COARSE_HISTORY:
            self._coarse_history_enqueue()
        P = [len(sq) for sq in self.seqs]
        self._check_room(max(P) + N)
        graphs = self.use_graphs and N == pol.draft_length
        if graphs:
            self._ensure_graphs()
            logits, draft_tok = self._step_graphed(P, N, ev1)
        else:
            # ---- drafting (eager)
            first = torch.tensor([[sq[-2], sq[-1]] for sq in self.seqs], dtype=torch.int64, device=dev)
            start = torch.tensor([p - 2 for p in P], dtype=torch.int64, device=dev)
            drafts = []
            inp = first
            for d in range(N):
                logits = self._draft_forward(inp, start, max(P) + d, d)
                tok = K.argmax_rows(logits)
                drafts.append(tok)
                start = (start + inp.shape[1]) if d == 0 else start + 1
                inp = tok.long().view(B, 1)
            draft_tok = torch.stack(drafts, dim=1).contiguous()  # [B, N] int32
            ev1.record(st)
            # ---- verification (eager)
            if self.use_worker:
                self._drain()
            last = torch.tensor([[sq[-1]] for sq in self.seqs], dtype=torch.int64, device=dev)
            vtok = torch.cat([last, draft_tok.long()], dim=1)  # [B, N+1]
            vstart = torch.tensor([p - 1 for p in P], dtype=torch.int64, device=dev)
            s = self.scratch if B * (N + 1) <= self.scratch.T else self._prefill_scratch(B * (N + 1))
            logits = self._target_forward(vtok, vstart, max(P) + N, s)
        _, res = K.greedy_accept(logits.contiguous(), draft_tok)
        if self.record:
            self.captures.append({"accept_logits": logits.clone(), "draft": draft_tok.clone(), "res": res.clone()})
        ev2.record(st)
        res_h = res.cpu().tolist()  # syncs
        draft_h = draft_tok.cpu().tolist()
        emitted = []
        for b in range(B):
            acc, nxt = res_h[b]
            new = draft_h[b][:acc] + [nxt]
            if remaining is not None:
                new = new[: max(0, remaining[b])]
            self.seqs[b].extend(new)
            emitted.append(len(new))
            self.emitted_total += len(new)
            self.accepted_total += acc
        self.drafted_total += N * B
        if self.record_routing and self._iter_logits:
            # committed positions of this verify: rows 0..accepted of each
            # sequence (the last committed token and the accepted drafts)
            from .tracefile import softmax_rows

            lg = torch.stack(self._iter_logits[-a.num_layers:]).cpu().numpy()  # [L, B*(N+1), E]
            lg = lg.reshape(a.num_layers, B, N + 1, -1)
            for b in range(B):
                for t in range(min(res_h[b][0] + 1, emitted[b])):
                    self.trace_scores[b].append(softmax_rows(lg[:, b, t, :]))
            self._iter_logits = []
        self.iter_events.append((ev0, ev1, ev2))
        self.iter_records.append(
            IterationRecord(
                index=len(self.iter_records), start=0.0, draft_end=0.0, verify_end=0.0,
                position=P[0], drafted=N, accepted=res_h[0][0], emitted=emitted[0],
            )
        )
        return emitted

    def generate(self, prompts: torch.Tensor, max_new_tokens: int) -> SimReport:
        """Prefill, then SD iterations until every sequence has
        ``max_new_tokens`` new tokens; returns the SimReport."""
        self.prefill(prompts)
        torch.cuda.synchronize(self.device)
        t0 = time.perf_counter()
        remaining = [max_new_tokens] * self.batch
        while any(r > 0 for r in remaining):
            em = self.step(remaining)
            remaining = [r - e for r, e in zip(remaining, em)]
        torch.cuda.synchronize(self.device)
        wall = time.perf_counter() - t0
        return self.report(wall_s=wall)

    # -------------------------------------------------------------- report
    def timing_summary(self) -> dict:
        self._fold_events(force=True)
        draft = verify = 0.0
        iters = []
        t = 0.0
        for d, v in self._iters_done:
            draft += d
            verify += v
            iters.append((t, t + d, t + d + v))
            t += d + v
        stall = dict(self._stall_done)
        return {"draft_ms": draft, "verify_ms": verify, "stall_ms": stall, "iters": iters}

    def export_trace(self, path, seq: int = 0) -> int:
        """Write the real gating scores of sequence ``seq``'s committed tokens
        as a reference trace-v1 file (needs ``record_routing=True``);
        returns the token count."""
        from .tracefile import write_trace

        rows = self.trace_scores[seq]
        if not rows:
            raise ValueError("no routing recorded (construct the engine with record_routing=True)")
        write_trace(path, np.stack(rows), self.arch.name, self.arch.top_k, 0, self.policy.seed)
        return len(rows)

    def transfers(self) -> list[TransferRecord]:
        out = []
        for r in self.cache.transfer_log():
            if r["end_ms"] < 0:
                continue
            out.append(
                TransferRecord(
                    start=r["start_ms"] / 1e3,
                    end=r["end_ms"] / 1e3,
                    nbytes=r["n_experts"] * self.arch.expert_bytes,
                    kind=TransferKind.PREFETCH if r["kind"] == "prefetch" else TransferKind.ON_DEMAND,
                    layer=r["layer"],
                    experts=r["experts"],
                )
            )
        return out

    def report(self, wall_s: float | None = None) -> SimReport:
        ts = self.timing_summary()
        total_ms = ts["draft_ms"] + ts["verify_ms"]
        stall_total = ts["stall_ms"]["prefetch"] + ts["stall_ms"]["demand"]
        if total_ms > 0:
            breakdown = {
                "draft": ts["draft_ms"] / total_ms,
                "expert_load": stall_total / total_ms,
                "attention_and_other": (ts["verify_ms"] - stall_total) / total_ms,
            }
        else:
            breakdown = {"draft": 0.0, "expert_load": 0.0, "attention_and_other": 1.0}
        c = self.cache.counters()
        transfers = self.transfers()
        pre = [t for t in transfers if t.kind is TransferKind.PREFETCH]
        dem = [t for t in transfers if t.kind is TransferKind.ON_DEMAND]
        pre_ms = sum(t.duration for t in pre) * 1e3
        h2d_bytes = sum(t.nbytes for t in transfers)
        h2d_ms = sum(t.duration for t in transfers) * 1e3
        wire = self.cache.wire_bytes()
        wire_bytes = wire["prefetch"] + wire["demand"]
        # link occupancy: union of [start, last H2D done] over the transfers
        spans = sorted((r["start_ms"], r["copy_end_ms"]) for r in self.cache.transfer_log()
                       if r["copy_end_ms"] >= 0)
        link_ms, copy_ms, cur = 0.0, 0.0, None
        for a_, b_ in spans:
            copy_ms += b_ - a_
            if cur is None or a_ > cur[1]:
                if cur is not None:
                    link_ms += cur[1] - cur[0]
                cur = [a_, b_]
            else:
                cur[1] = max(cur[1], b_)
        if cur is not None:
            link_ms += cur[1] - cur[0]
        iters = [
            IterationRecord(r.index, it[0] / 1e3, it[1] / 1e3, it[2] / 1e3, r.position, r.drafted, r.accepted, r.emitted)
            for r, it in zip(self.iter_records, ts["iters"])
        ]
        # compute slots on the same clock as the transfer log (runtime epoch)
        self._fold_events(force=True)
        slots = list(self._slots_done)
        n_emit = self.emitted_total
        extras = {
            "batch": self.batch,
            "acceptance_rate": (self.accepted_total / self.drafted_total) if self.drafted_total else 0.0,
            "mean_accepted_per_iter": (self.accepted_total / len(self.iter_records)) if self.iter_records else 0.0,
            "stall_prefetch_ms": ts["stall_ms"]["prefetch"],
            "stall_demand_ms": ts["stall_ms"]["demand"],
            "prefetch_copy_ms": pre_ms,
            "hidden_prefetch_fraction": (1.0 - ts["stall_ms"]["prefetch"] / pre_ms) if pre_ms > 0 else None,
            "h2d_bytes": h2d_bytes,
            # expert bytes made resident per second of copy time (decoded)
            "h2d_gbs": (h2d_bytes / (h2d_ms / 1e3) / 1e9) if h2d_ms > 0 else None,
            "host_codec": self.host_pool.codec,
            "h2d_wire_bytes": wire_bytes,
            # bytes that crossed the host link per second of copy time
            "h2d_wire_gbs": (wire_bytes / (copy_ms / 1e3) / 1e9) if copy_ms > 0 else None,
            # time the host link was copying, and as a fraction of device time
            "link_busy_ms": link_ms,
            "link_busy_frac": (link_ms / total_ms) if total_ms > 0 else None,
            "h2d_wire_ratio": (wire_bytes / h2d_bytes) if h2d_bytes else None,
            "n_prefetch_transfers": len(pre),
            "n_demand_transfers": len(dem),
            "wall_s": wall_s,
            "tokens_per_s": n_emit / (total_ms / 1e3) if total_ms > 0 else 0.0,
            "device_ms": total_ms,
        }
        counters = {k_: c[k_] for k_ in (
            "hits", "misses", "evictions", "prefetch_insertions", "prefetch_evictions",
            "demand_insertions", "tasks_completed", "tasks_aborted", "evictions_of_queued_targets")}
        return SimReport(
            policy=self.policy,
            seed=self.policy.seed,
            tpot=(total_ms / 1e3) / n_emit if n_emit else 0.0,
            hit_rate=self.cache.hit_rate(),
            eviction_rate=self.cache.eviction_rate(),
            latency_breakdown=breakdown,
            total_time=total_ms / 1e3,
            emitted_tokens=n_emit,
            cutoff_effective=self.cutoff,
            cache_capacity=self.capacity,
            iterations=iters,
            transfers=transfers,
            compute_slots=slots,
            counters=counters,
            extras=extras,
        )


def simulate(model, hw, timings, policy, trace=None, predictor=None, warm_start=False, *, arch=None,
             prompts=None, max_new_tokens: int = 32, batch: int = 1, **engine_kw) -> SimReport:
    """``moesim.simulate``-shaped entry point running the real B200 engine.

    ``trace`` and ``predictor`` must be None: routing and prediction come from
    the model's hidden states (the draft-guided predictor).  ``arch`` gives
    the shapes (default: inferred preset by name, else 'tiny')."""
    from .model import ARCH_PRESETS

    if trace is not None or predictor is not None:
        raise ValidationError("the B200 engine computes routing from hidden states; pass trace=None")
    if arch is None:
        arch = ARCH_PRESETS.get(getattr(model, "name", ""), ARCH_PRESETS["tiny"])
    eng = SpecMoEEngine(arch, hw, timings, policy, batch=batch, **engine_kw)
    try:
        if prompts is None:
            g = torch.Generator().manual_seed(policy.seed)
            prompts = torch.randint(0, arch.vocab, (batch, 16), generator=g)
        return eng.generate(prompts, max_new_tokens)
    finally:
        eng.close()


def _run_points(model, hw, timings, policies, *, arch=None, prompts=None, max_new_tokens: int = 32, batch: int = 1,
                **engine_kw) -> list[SimReport]:
    """One engine per policy over ONE model build (pinned host pool and
    device weights shared through ``model_state``) and identical prompts."""
    from .model import ARCH_PRESETS

    if arch is None:
        arch = ARCH_PRESETS.get(getattr(model, "name", ""), ARCH_PRESETS["tiny"])
    owner = None
    shared = engine_kw.pop("model_state", None)  # a caller-owned model build
    out = []
    try:
        for p in policies:
            if prompts is None:
                g = torch.Generator().manual_seed(p.seed)
                prompts = torch.randint(0, arch.vocab, (batch, 16), generator=g)
            state = shared if shared is not None else (owner.model_state if owner is not None else None)
            kw = dict(engine_kw)
            kw.setdefault("max_tokens", max(prompts.shape[1] + max_new_tokens + 8, 64))
            eng = SpecMoEEngine(arch, hw, timings, p, batch=batch, model_state=state, **kw)
            try:
                out.append(eng.generate(prompts, max_new_tokens))
            finally:
                if owner is None and shared is None:
                    owner = eng  # keeps the shared model alive until the last point
                else:
                    eng.close()
    finally:
        if owner is not None:
            owner.close()
    return out


def compare_policies(model, hw, timings, policies, trace=None, warm_start=False, *, arch=None, prompts=None,
                     max_new_tokens: int = 32, batch: int = 1, **engine_kw) -> list[SimReport]:
    """``moesim.compare_policies`` (``simcore.py:518-527``) on the real
    engine: one report per policy over the identical model, prompts and seed.

    ``trace`` must be None (routing comes from the hidden states).  The
    engine's prefill always leaves the prompt's experts resident, which is
    the real-run counterpart of the reference's ``warm_start`` fill
    (``simcore.py:299-307``); ``warm_start`` is accepted for signature
    compatibility."""
    if trace is not None:
        raise ValidationError("the B200 engine computes routing from hidden states; pass trace=None")
    if not policies:
        return []
    return _run_points(model, hw, timings, list(policies), arch=arch, prompts=prompts,
                       max_new_tokens=max_new_tokens, batch=batch, **engine_kw)


SWEEP_PARAMETERS = {
    "cutoff_layer": "cutoff_layer",
    "draft_length": "draft_length",
    "cache_capacity": "cache_capacity_experts",
    "prefetch_k": "prefetch_k",
}


def sweep(parameter: str, values: list, model, hw, timings, policy, trace=None, warm_start=False, *, arch=None,
          prompts=None, max_new_tokens: int = 32, batch: int = 1, **engine_kw) -> list[tuple[object, SimReport]]:
    """``moesim.sweep`` (``simcore.py:530-564``) on the real engine: one run
    per parameter value, same model build, prompts and seed; same parameter
    names and the same ValidationError rules as the reference."""
    from dataclasses import replace

    if parameter not in SWEEP_PARAMETERS:
        raise ValidationError(f"unknown sweep parameter {parameter!r}; choose from {sorted(SWEEP_PARAMETERS)}")
    if not values:
        raise ValidationError("sweep range is empty")
    if parameter == "cutoff_layer" and policy.policy is not Policy.DRAFT_PREFETCH:
        raise ValidationError("cutoff_layer sweeps require the draft_prefetch policy")
    if parameter == "prefetch_k" and policy.policy is Policy.ON_DEMAND:
        raise ValidationError("prefetch_k does not apply to the on_demand policy")
    if trace is not None:
        raise ValidationError("the B200 engine computes routing from hidden states; pass trace=None")
    field_name = SWEEP_PARAMETERS[parameter]
    pols = [replace(policy, **{field_name: int(v)}) for v in values]
    reps = _run_points(model, hw, timings, pols, arch=arch, prompts=prompts, max_new_tokens=max_new_tokens,
                       batch=batch, **engine_kw)
    return list(zip(values, reps))
