"""The SP-MoE draft/verify SD loop on the host cores.

TEST INFRASTRUCTURE ONLY (see spmoe_oracle.c): the oracle of the whole
speculative-decoding loop for the end-to-end parity tests, and the CPU
restatement that bench.py times as the reference arm / cpu_baseline.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs import it.

It mirrors ``SpecMoEEngine`` step for step on the same determinism contract:

* ``prefill``: draft and target forwards over ``prompt[:-1]`` from position 0;
* ``step`` (``Simulation.run`` / ``_draft_stage`` / ``_verify_stage`` of
  simcore.py:323-465 with real tensors): N draft steps -- the first over the
  last two committed tokens at position P-2, then one token each -- with the
  draft-guided predictor (K1 on the draft's layer-l MLP input against target
  router l, Algorithm 1) at layers <= cutoff; then the
  verify pass over ``[last, d_0..d_{N-1}]`` at position P-1 through the
  target MoE (K1 top-k, K2 permute, K3 SwiGLU experts, K4 combine of Eq. 1,
  PAPER.md:170-175); then greedy acceptance (longest matching prefix plus the
  correction/bonus token; the deterministic counterpart of
  simcore.py:440-446).

Every op is a C oracle function (oracle/cpu_path.c on lane-major weights,
forward_oracle.c, spmoe_oracle.c).  Weights come either from a GPU engine
(:meth:`CpuWeights.from_engine`, the parity tests) or from the CPU
restatement of the counter-hash init (:meth:`CpuWeights.generate`, the
reference arm: no GPU involved).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import tensor_oracle as O

MASK64 = (1 << 64) - 1
# kind codes of the counter-hash init (model.tensor_seed; checked equal in
# tests/test_cpu_path.py)
K_EMBED, K_QKV, K_WO, K_ROUTER, K_EXPERT, K_SHARED, K_SGATE, K_LMHEAD, K_PERTURB, K_BASE = range(10)
ONE_BF16 = 0x3F80


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def tensor_seed(base: int, *ids: int) -> int:
    h = splitmix64(base & MASK64)
    for v in ids:
        h = splitmix64(h ^ (v & MASK64))
    return h


def rope_tables(head_dim: int, theta: float, max_seq: int) -> tuple[np.ndarray, np.ndarray]:
    """Rotate-half tables from libm doubles rounded to f32 (the model's
    rope_tables_host; equality checked in tests)."""
    inv = [1.0 / (theta ** (i / head_dim)) for i in range(0, head_dim, 2)]
    cos = np.empty((max_seq, head_dim), np.float32)
    sin = np.empty((max_seq, head_dim), np.float32)
    for p in range(max_seq):
        c = [math.cos(p * f) for f in inv]
        s = [math.sin(p * f) for f in inv]
        cos[p] = c + c
        sin[p] = s + s
    return cos, sin


def gate_mass(router: np.ndarray, top_k: int, renorm: bool) -> float:
    """Expected routed gate mass (model.gate_mass, restated)."""
    if renorm:
        return 1.0
    xs = np.random.default_rng(0).standard_normal((512, router.shape[1]))
    lg = xs @ router.astype(np.float64).T
    p = np.exp(lg - lg.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    return float(np.sort(p, axis=-1)[:, -top_k:].sum(-1).mean())


@dataclass
class Arch:
    """The shape fields the forward needs (duck-typed from model.ArchSpec)."""

    vocab: int
    hidden: int
    num_layers: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    num_experts: int
    top_k: int
    renorm: bool
    shared_ffn: int
    shared_gate: bool
    d_ffn: int
    rope_theta: float
    rms_eps: float
    max_seq: int

    @classmethod
    def of(cls, a) -> "Arch":
        return cls(**{f: getattr(a, f) for f in cls.__dataclass_fields__})


@dataclass
class CpuLayer:
    attn_norm: np.ndarray
    wqkv: np.ndarray  # LM [qkv, Hp]
    wo: np.ndarray  # LM [H, (nh*hd)p]
    ffn_norm: np.ndarray
    router: np.ndarray  # raw [E, H]
    draft: np.ndarray  # LM blob (d_ffn)
    shared: np.ndarray | None = None  # LM blob (shared_ffn)
    sgate: np.ndarray | None = None  # raw [H]


@dataclass
class CpuWeights:
    arch: Arch
    embed: np.ndarray  # raw [V, H]
    lm_head: np.ndarray  # LM [V, Hp]
    final_norm: np.ndarray
    layers: list[CpuLayer]
    cos: np.ndarray
    sin: np.ndarray
    expert: Callable[[int, int], np.ndarray] = None  # (layer, e) -> LM blob
    experts: dict = field(default_factory=dict)

    # ------------------------------------------------------------ builders
    @classmethod
    def from_engine(cls, eng, raw_expert: Callable[[int, int], np.ndarray], cache_layers: int = 2) -> "CpuWeights":
        """Copy a GPU engine's device weights (bits) into lane-major host
        arrays; routed experts are fetched lazily through ``raw_expert(l, e)``
        (raw bf16 bits of the host-pool row), packed, and kept for the last
        ``cache_layers`` layers."""
        import torch

        def bits(t):
            return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)

        a = Arch.of(eng.arch)
        w = eng.weights
        H = a.hidden
        layers = []
        for lw in w.layers:
            layers.append(CpuLayer(
                attn_norm=bits(lw.attn_norm), wqkv=O.pack_lm(bits(lw.wqkv)), wo=O.pack_lm(bits(lw.wo)),
                ffn_norm=bits(lw.ffn_norm), router=bits(lw.router),
                draft=O.pack_blob(bits(lw.draft_ffn[0]), H, a.d_ffn),
                shared=None if lw.shared is None else O.pack_blob(bits(lw.shared[0]), H, a.shared_ffn),
                sgate=None if lw.shared_gate is None else bits(lw.shared_gate)))
        cw = cls(arch=a, embed=bits(w.embed), lm_head=O.pack_lm(bits(w.lm_head)), final_norm=bits(w.final_norm),
                 layers=layers, cos=w.rope_cos.cpu().numpy(), sin=w.rope_sin.cpu().numpy())
        order: list[int] = []

        def expert(l, e):
            key = (l, e)
            if key not in cw.experts:
                if l not in order:
                    order.append(l)
                    while len(order) > cache_layers:
                        old = order.pop(0)
                        for k in [k for k in cw.experts if k[0] == old]:
                            del cw.experts[k]
                cw.experts[key] = O.pack_blob(raw_expert(l, e), H, a.ffn)
            return cw.experts[key]

        cw.expert = expert
        return cw

    @classmethod
    def generate(cls, arch, seed: int, log=None) -> "CpuWeights":
        """The counter-hash init of model.build_weights restated on the host
        (no GPU): every tensor bit-identical to the engine's (raw host-pool
        rows l*E+e; no draft perturbation)."""
        a = Arch.of(arch)
        H, E, F = a.hidden, a.num_experts, a.ffn
        std = float(arch.init_std)
        res_scale = float(arch.res_scale)
        out_scale = float(arch.expert_out_scale) * res_scale
        lib = O.lib()
        n13 = F * H

        def fill(n, s, sd):
            return O.fill_normal_bf16(n, s, 0, sd)

        def blob_generic(Fx, s, sd, osc):
            m = Fx * H
            b = np.empty(3 * m, np.uint16)
            b[:m] = fill(m, splitmix64(s ^ 1), sd)
            b[m:2 * m] = fill(m, splitmix64(s ^ 3), sd)
            b[2 * m:] = fill(m, splitmix64(s ^ 2), sd * osc)
            return b

        embed = fill(a.vocab * H, tensor_seed(seed, K_EMBED), float(arch.embed_std)).reshape(a.vocab, H)
        lm_head = O.pack_lm(fill(a.vocab * H, tensor_seed(seed, K_LMHEAD), std).reshape(a.vocab, H))
        ones = np.full((H,), ONE_BF16, np.uint16)
        experts: dict = {}
        layers = []
        qkv_dim = (a.num_heads + 2 * a.num_kv_heads) * a.head_dim
        for l in range(a.num_layers):
            wqkv = fill(qkv_dim * H, tensor_seed(seed, K_QKV, l), std).reshape(qkv_dim, H)
            wo = fill(H * a.num_heads * a.head_dim, tensor_seed(seed, K_WO, l), std * res_scale).reshape(
                H, a.num_heads * a.head_dim)
            router = fill(E * H, tensor_seed(seed, K_ROUTER, l), 1.0 / math.sqrt(H)).reshape(E, H)
            base = None
            if arch.expert_spread is not None:
                base = blob_generic(F, tensor_seed(seed, K_BASE, l), std, out_scale)
            acc = np.zeros(3 * n13, np.float32)
            for e in range(E):
                raw = blob_generic(F, tensor_seed(seed, K_EXPERT, l * E + e), std, out_scale)
                if base is not None:
                    lib.cpu_upcycle(base.ctypes.data, raw.ctypes.data, raw.size, float(arch.expert_spread))
                lib.cpu_accum(acc.ctypes.data, raw.ctypes.data, raw.size)
                experts[(l, e)] = O.pack_blob(raw, H, F)
                del raw
            mean = np.empty(3 * n13, np.uint16)
            lib.cpu_div_bf16(acc.ctypes.data, acc.size, float(E), mean.ctypes.data)
            del acc, base
            shared = sgate = None
            if a.shared_ffn:
                shared = blob_generic(a.shared_ffn, tensor_seed(seed, K_SHARED, l), std, out_scale)
                if a.shared_gate:
                    sgate = fill(H, tensor_seed(seed, K_SGATE, l), 1.0 / math.sqrt(H))
            if arch.draft_ffn:
                draft = blob_generic(a.d_ffn, tensor_seed(seed, K_EXPERT, l, 10_000), std, out_scale)
            else:
                draft = _draft_proxy(a, mean, shared, router)
            layers.append(CpuLayer(
                attn_norm=ones, wqkv=O.pack_lm(wqkv), wo=O.pack_lm(wo), ffn_norm=ones, router=router,
                draft=O.pack_blob(draft, H, a.d_ffn),
                shared=None if shared is None else O.pack_blob(shared, H, a.shared_ffn), sgate=sgate))
            if log:
                log(f"[cpu] generated layer {l + 1}/{a.num_layers}")
        cos, sin = rope_tables(a.head_dim, a.rope_theta, a.max_seq)
        cw = cls(arch=a, embed=embed, lm_head=lm_head, final_norm=ones, layers=layers, cos=cos, sin=sin,
                 experts=experts)
        cw.expert = lambda l, e: cw.experts[(l, e)]
        return cw


def _draft_proxy(a: Arch, mean: np.ndarray, shared: np.ndarray | None, router: np.ndarray) -> np.ndarray:
    """model._draft_proxy restated: mean routed expert with W2 scaled by the
    gate mass, concatenated along F with the shared expert (not with a
    sigmoid-gated one: the draft runs it beside, CpuSD._draft_ffn)."""
    H, F = a.hidden, a.ffn
    mass = gate_mass(O.bf16_bits_to_f32(router), a.top_k, a.renorm)
    w1 = mean[: F * H].reshape(F, H)
    w3 = mean[F * H: 2 * F * H].reshape(F, H)
    w2 = mean[2 * F * H:].reshape(H, F).copy()
    if mass != 1.0:
        O.lib().cpu_scale_bf16(w2.ctypes.data, w2.size, float(mass))
    if shared is None or a.shared_gate:
        return np.concatenate([w1.reshape(-1), w3.reshape(-1), w2.reshape(-1)])
    Fs = a.shared_ffn
    s1 = shared[: Fs * H].reshape(Fs, H)
    s3 = shared[Fs * H: 2 * Fs * H].reshape(Fs, H)
    s2 = shared[2 * Fs * H:].reshape(H, Fs)
    d1 = np.concatenate([w1, s1], axis=0)
    d3 = np.concatenate([w3, s3], axis=0)
    d2 = np.concatenate([w2, s2], axis=1)
    return np.concatenate([d1.reshape(-1), d3.reshape(-1), d2.reshape(-1)])


class CpuSD:
    """SpecMoEEngine's SD loop on the host cores (see module docstring)."""

    def __init__(self, w: CpuWeights, batch: int, N: int, kv_max_seq: int, cutoff: int | None = None,
                 prefetch_k: int = 1, predict: bool = True):
        a = w.arch
        self.w, self.a, self.B, self.N = w, a, batch, N
        self.cutoff, self.pk, self.predict = cutoff, prefetch_k, predict
        self.S = kv_max_seq
        shape = (a.num_layers, batch, a.num_kv_heads, self.S, a.head_dim)
        self.dk, self.dv = np.zeros(shape, np.uint16), np.zeros(shape, np.uint16)
        self.tk, self.tv = np.zeros(shape, np.uint16), np.zeros(shape, np.uint16)
        self.scale = float(a.head_dim ** -0.5)
        self.lib = O.lib()
        self.predictions: list = []  # (step, layer, idx) of the drafting-stage predictor
        self.logits: list = []  # verify logits per iteration (record=True)
        self.record = False

    # ---------------------------------------------------------- forwards
    def _attn(self, l: int, x: np.ndarray, T: int, start: np.ndarray, kc, vc) -> None:
        a, lw = self.a, self.w.layers[l]
        self.lib.cpu_attn_block(
            x.ctypes.data, self.B, T, a.hidden, lw.wqkv.ctypes.data, lw.wo.ctypes.data, lw.attn_norm.ctypes.data,
            a.rms_eps, a.num_heads, a.num_kv_heads, a.head_dim, self.w.cos.ctypes.data, self.w.sin.ctypes.data,
            self.w.cos.shape[0], start.ctypes.data, kc[l].ctypes.data, vc[l].ctypes.data, self.S, self.scale)

    def _dense(self, blob: np.ndarray, F: int, hn: np.ndarray, x: np.ndarray) -> np.ndarray:
        n = hn.shape[0]
        _, y = O.lm_expert_ffn(blob, self.a.hidden, F, hn, n=n)
        return O.moe_combine(y, np.arange(n, dtype=np.int32), None, n, self.a.hidden, 1, residual=x)

    def _draft_ffn(self, l: int, hn: np.ndarray, x: np.ndarray) -> np.ndarray:
        """engine._draft_ffn restated: the dense FFN, or for a sigmoid-gated
        shared expert the mean-expert FFN + the gated shared expert (K4)."""
        a, lw = self.a, self.w.layers[l]
        if not (a.shared_gate and lw.shared is not None and lw.sgate is not None):
            return self._dense(lw.draft, a.d_ffn, hn, x)
        n = hn.shape[0]
        _, y = O.lm_expert_ffn(lw.draft, a.hidden, a.d_ffn, hn, n=n)
        _, ys = O.lm_expert_ffn(lw.shared, a.hidden, a.shared_ffn, hn, n=n)
        _, _, _, sg = O.router_topk(hn, lw.router, 1, a.renorm, lw.sgate)
        return O.moe_combine(y, np.arange(n, dtype=np.int32), None, n, a.hidden, 1, ys=ys, sg=sg, residual=x)

    def draft_forward(self, tokens: np.ndarray, start: np.ndarray, step: int | None) -> np.ndarray:
        """tokens [B, T] -> last-token logits [B, V] f32 (draft KV appended)."""
        a, w = self.a, self.w
        B, T = tokens.shape
        x = np.ascontiguousarray(w.embed[tokens.reshape(-1)])
        for l in range(a.num_layers):
            lw = w.layers[l]
            self._attn(l, x, T, start, self.dk, self.dv)
            hn = O.rms_norm(x, lw.ffn_norm, a.rms_eps)
            if step is not None and self.predict and self.cutoff is not None and l <= self.cutoff:
                last = hn.reshape(B, T, -1)[:, -1, :]
                _, idx, _, _ = O.router_topk(last, lw.router, self.pk, True)
                self.predictions.append((step, l, idx))
            x = self._draft_ffn(l, hn, x)
        last = np.ascontiguousarray(x.reshape(B, T, -1)[:, -1, :])
        return O.lm_linear(w.lm_head, a.hidden, last, norm_w=w.final_norm, eps=a.rms_eps, f32=True)

    def moe(self, l: int, hn: np.ndarray, x: np.ndarray) -> np.ndarray:
        """Verify-MoE layer l: K1, K2, K3 over the routed experts, shared
        expert, K4 combine with the residual."""
        a, lw = self.a, self.w.layers[l]
        T, H = hn.shape
        k, E = a.top_k, a.num_experts
        wts, idx, _, sg = O.router_topk(hn, lw.router, k, a.renorm, lw.sgate)
        off, perm, inv = O.moe_permute(idx, E)
        y = np.zeros((T * k, H), np.float32)
        for e in range(E):
            o0, o1 = int(off[e]), int(off[e + 1])
            if o1 > o0:
                _, y[o0:o1] = O.lm_expert_ffn(self.w.expert(l, e), H, a.ffn, hn, perm[o0:o1])
        ys = None
        if lw.shared is not None:
            _, ys = O.lm_expert_ffn(lw.shared, H, a.shared_ffn, hn, n=T)
        return O.moe_combine(y, inv, wts, T, H, k, ys=ys, sg=sg, residual=x)

    def target_forward(self, tokens: np.ndarray, start: np.ndarray, logits: bool = True) -> np.ndarray | None:
        """tokens [B, T] -> logits [B, T, V] f32 (target KV appended)."""
        a, w = self.a, self.w
        B, T = tokens.shape
        x = np.ascontiguousarray(w.embed[tokens.reshape(-1)])
        for l in range(a.num_layers):
            lw = w.layers[l]
            self._attn(l, x, T, start, self.tk, self.tv)
            hn = O.rms_norm(x, lw.ffn_norm, a.rms_eps)
            x = self.moe(l, hn, x)
        if not logits:
            return None
        lg = O.lm_linear(w.lm_head, a.hidden, x, norm_w=w.final_norm, eps=a.rms_eps, f32=True)
        return lg.reshape(B, T, -1)

    # ------------------------------------------------------------ SD loop
    def prefill(self, prompts: np.ndarray) -> None:
        prompts = np.asarray(prompts, np.int64)
        B, P = prompts.shape
        if B != self.B or P < 2 or P > self.S:
            raise ValueError("prompts must be [batch, 2..kv_max_seq]")
        self.seqs = [list(map(int, r)) for r in prompts]
        ctx = np.ascontiguousarray(prompts[:, :-1])
        z = np.zeros((B,), np.int64)
        self.draft_forward(ctx, z, None)
        self.target_forward(ctx, z, logits=False)

    def step(self, remaining: list[int] | None = None) -> list[int]:
        """One SD iteration; returns tokens emitted per sequence."""
        B, N = self.B, self.N
        if remaining is not None and B == 1:
            N = max(1, min(N, remaining[0]))
        P = [len(s) for s in self.seqs]
        if max(P) + N > self.S:
            raise ValueError("KV caches full")
        inp = np.array([[s[-2], s[-1]] for s in self.seqs], np.int64)
        start = np.array([p - 2 for p in P], np.int64)
        drafts = []
        for d in range(N):
            lg = self.draft_forward(inp, start, d)
            tok = O.argmax_rows(lg)
            drafts.append(tok)
            start = start + (inp.shape[1] if d == 0 else 1)
            inp = tok.astype(np.int64).reshape(B, 1)
        draft = np.stack(drafts, axis=1).astype(np.int32)  # [B, N]
        vtok = np.concatenate([np.array([[s[-1]] for s in self.seqs], np.int64), draft.astype(np.int64)], axis=1)
        vstart = np.array([p - 1 for p in P], np.int64)
        logits = self.target_forward(vtok, vstart)
        _, res = O.greedy_accept(logits, draft)
        if self.record:
            self.logits.append((logits, draft, res))
        emitted = []
        for b in range(B):
            acc, nxt = int(res[b, 0]), int(res[b, 1])
            new = [int(t) for t in draft[b, :acc]] + [nxt]
            if remaining is not None:
                new = new[: max(0, remaining[b])]
            self.seqs[b].extend(new)
            emitted.append(len(new))
        return emitted
