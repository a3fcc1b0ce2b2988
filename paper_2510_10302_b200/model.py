"""Model shapes, deterministic random weights, the pinned host expert pool and
the non-MoE transformer pieces of the draft/target pair.

The reference simulates model behaviour with activation traces
(``trace.py:103-173``); the B200 build runs real (random-init) weights of the
named shapes so that routing, prediction and acceptance come out of actual
hidden states.  Everything here is plumbing around the hot path:

* :class:`ArchSpec` — hidden size, heads, expert width ... plus presets for
  the BASELINE.json configs (tiny, Mixtral-8x7B, DeepSeek-V2-Lite,
  Qwen1.5-MoE-A2.7B).  Attention is standard GQA/MHA for every preset (the
  verify-time expert path does not depend on DeepSeek's MLA).
* :class:`HostExpertPool` — every routed expert of every layer as one
  contiguous bf16 blob ``W1[F,H] | W3[F,H] | W2[H,F]`` in page-locked host
  memory (the offload tier), generated on the GPU with the counter-hash init
  and copied down.
* :class:`ModelWeights` — device-resident embedding, attention, norms, router,
  shared experts, lm_head, and the draft's dense FFN.  The draft shares the
  target's embedding, attention and lm_head (SURVEY.md §7 hard part 2) and
  uses the mean of the layer's experts as its FFN, optionally perturbed.
* the attention block and lm_head around the MoE: K9 fixed-order
  projections, RoPE + KV append and attention kernels (csrc/spmoe_attn.cu),
  all inside the determinism contract so the whole forward is reproducible
  on the CPU oracle.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import asdict, dataclass, replace
from pathlib import Path

import numpy as np
import torch
import yaml

from .config import ModelSpec, ValidationError

MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------------------
# shapes
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ArchSpec:
    name: str
    vocab: int
    hidden: int
    num_layers: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int  # routed expert intermediate size
    num_experts: int  # routed experts per layer
    top_k: int
    renorm: bool = True  # Mixtral: renormalise top-k; DeepSeek/Qwen: no
    shared_ffn: int = 0  # total intermediate size of the shared expert(s)
    shared_gate: bool = False  # Qwen1.5-MoE sigmoid gate on the shared expert
    draft_ffn: int = 0  # draft dense FFN width (0 -> ffn)
    rope_theta: float = 1e6
    rms_eps: float = 1e-5
    max_seq: int = 2048
    init_std: float = 0.02
    expert_out_scale: float = 1.0  # scales W2 std (residual-branch scaling)
    # Upcycled experts (None = independent random experts): every routed
    # expert of a layer = shared layer component + expert_spread x its own
    # deviation, so the draft's mean-expert FFN tracks the routed mixture and
    # random-init SD accepts drafts at a realistic rate (SURVEY.md §7 hard
    # part 2).  Bytes moved and FLOPs are unchanged.
    expert_spread: float | None = 0.02
    # init scales: token embedding std, and GPT-2-style residual-branch
    # scaling of the output projections (W_o, W2): std * residual_scale,
    # None -> 1/sqrt(2 * num_layers).  Keeps the 32-layer random network out
    # of the chaotic regime so a slightly different draft still agrees.
    embed_std: float = 1.0
    residual_scale: float | None = None

    @property
    def res_scale(self) -> float:
        return self.residual_scale if self.residual_scale is not None else 1.0 / math.sqrt(2 * self.num_layers)

    def __post_init__(self):
        if self.hidden % 8 or self.ffn % 8 or (self.shared_ffn % 8):
            raise ValidationError("hidden and ffn sizes must be multiples of 8")
        if not 1 <= self.top_k <= self.num_experts <= 64:
            raise ValidationError("need 1 <= top_k <= num_experts <= 64")
        if self.num_heads % self.num_kv_heads:
            raise ValidationError("num_heads must be a multiple of num_kv_heads")

    @property
    def expert_elems(self) -> int:
        return 3 * self.ffn * self.hidden

    @property
    def expert_bytes(self) -> int:
        return 2 * self.expert_elems

    @property
    def d_ffn(self) -> int:
        """Draft dense FFN width: explicit, else the derived proxy (mean routed
        expert, plus the shared expert(s) concatenated along F -- unless the
        shared expert is sigmoid-gated: then the draft runs the target's
        shared expert and gate beside the mean expert, see _draft_proxy)."""
        return self.draft_ffn or (self.ffn + (0 if self.shared_gate else self.shared_ffn))

    @property
    def qkv_dim(self) -> int:
        return (self.num_heads + 2 * self.num_kv_heads) * self.head_dim


ARCH_PRESETS: dict[str, ArchSpec] = {
    # BASELINE config #1: tiny Mixtral-style target (4 layers, 8 experts top-2,
    # hidden 256); vocab kept small so the CPU oracle finishes in seconds.
    "tiny": ArchSpec(
        name="tiny", vocab=512, hidden=256, num_layers=4, num_heads=4, num_kv_heads=2,
        head_dim=64, ffn=512, num_experts=8, top_k=2, max_seq=512,
    ),
    # BASELINE config #2: Mixtral-8x7B shapes (HF config)
    "mixtral_8x7b": ArchSpec(
        name="mixtral_8x7b", vocab=32000, hidden=4096, num_layers=32, num_heads=32,
        num_kv_heads=8, head_dim=128, ffn=14336, num_experts=8, top_k=2, rope_theta=1e6,
        max_seq=1024,
        # measured acceptance vs spread (profiles/r1_acceptance_spread.jsonl,
        # 20 SD iterations x 2 prompts): 0.02 -> 0.83-0.90, 0.005 -> 0.94-0.96,
        # the paper's ~97 %
        expert_spread=0.005,
    ),
    # BASELINE config #3: DeepSeek-V2-Lite MoE shapes (64 routed + 2 shared of
    # 1408, top-6, no top-k renorm); 27 MoE layers as in the reference ModelSpec
    "deepseek_v2_lite": ArchSpec(
        name="deepseek_v2_lite", vocab=102400, hidden=2048, num_layers=27, num_heads=16,
        num_kv_heads=16, head_dim=128, ffn=1408, num_experts=64, top_k=6, renorm=False,
        shared_ffn=2 * 1408, rope_theta=1e4, rms_eps=1e-6, max_seq=1024,
    ),
    # BASELINE config #4: Qwen1.5-MoE-A2.7B shapes (60 routed top-4, shared
    # expert 5632 with sigmoid gate)
    "qwen15_moe_a27b": ArchSpec(
        name="qwen15_moe_a27b", vocab=151936, hidden=2048, num_layers=24, num_heads=16,
        num_kv_heads=16, head_dim=128, ffn=1408, num_experts=60, top_k=4, renorm=False,
        shared_ffn=5632, shared_gate=True, rope_theta=1e6, rms_eps=1e-6, max_seq=1024,
    ),
}


def get_arch(name_or_spec, **overrides) -> ArchSpec:
    a = ARCH_PRESETS[name_or_spec] if isinstance(name_or_spec, str) else name_or_spec
    return replace(a, **overrides) if overrides else a


def load_arch(path: str | Path) -> ArchSpec | None:
    """The optional ``arch`` section of an experiment file (None if absent).
    ``arch: {preset: mixtral_8x7b, ...overrides}`` or a full field list."""
    doc = yaml.safe_load(Path(path).read_text())
    sec = (doc or {}).get("arch")
    if sec is None:
        return None
    sec = dict(sec)
    preset = sec.pop("preset", None)
    if preset is not None:
        return get_arch(preset, **sec)
    return ArchSpec(**sec)


def model_spec_for(arch: ArchSpec, draft_layers: int | None = None) -> ModelSpec:
    """The reference ModelSpec of an arch (routed experts only: shared experts
    stay resident outside the cache budget, SURVEY.md §7 hard part 8)."""
    return ModelSpec(
        name=arch.name,
        num_layers=arch.num_layers,
        experts_per_layer=arch.num_experts,
        topk_activated=arch.top_k,
        shared_experts=0,
        expert_size=arch.expert_bytes,
        draft_layers=draft_layers or arch.num_layers,
        draft_topk=0,
    )


def arch_dict(arch: ArchSpec) -> dict:
    return asdict(arch)


# ---------------------------------------------------------------------------
# deterministic init
# ---------------------------------------------------------------------------
def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def tensor_seed(base: int, *ids: int) -> int:
    """64-bit seed of one named tensor (ids: kind code, layer, expert ...)."""
    h = _splitmix64(base & MASK64)
    for v in ids:
        h = _splitmix64(h ^ (v & MASK64))
    return h


# kind codes for tensor_seed
K_EMBED, K_QKV, K_WO, K_ROUTER, K_EXPERT, K_SHARED, K_SGATE, K_LMHEAD, K_PERTURB, K_BASE = range(10)


# ---------------------------------------------------------------------------
# host expert pool
# ---------------------------------------------------------------------------
class HostExpertPool:
    """Page-locked host memory holding every routed expert blob.

    ``index[l*E + e]`` is the pool row of expert (l, e); with ``distinct`` <
    L*E rows, experts alias rows (bounded host RAM; the bytes moved per copy
    are unchanged).  Allocated with cudaHostAlloc (exact size, portable,
    mapped) through the native library.

    ``codec="xc"``: rows hold XC blobs (codec.py) instead of raw bf16; the
    row stride is the largest blob, known only after the experts exist, so
    :func:`build_weights` sizes the blobs first and then calls
    :meth:`allocate`.
    """

    def __init__(self, arch: ArchSpec, distinct: int | None = None, share: str | None = None,
                 leader: bool = True, codec: str | None = None):
        """``share`` = name of a /dev/shm pool shared by the per-GPU processes
        of one box (replica mode): the local leader creates and fills it
        (``writable``), followers attach once the leader publishes it."""
        from . import _native

        if codec not in (None, "xc"):
            raise ValueError("codec must be None or 'xc'")
        self.arch = arch
        n = arch.num_layers * arch.num_experts
        self.rows = n if not distinct else min(int(distinct), n)
        self.index = [i % self.rows for i in range(n)]
        self.slot_bytes = arch.expert_bytes
        self.codec = codec
        self._lib = _native.load()
        self._shared = None
        self._share = share
        self.writable = leader
        self.ptr = None
        self.row_stride = 0
        self.wire = [arch.expert_bytes] * self.rows  # bytes of each row that cross the link
        if codec is None:
            self.allocate(arch.expert_bytes)

    def allocate(self, row_stride: int) -> None:
        """Back the pool with ``rows * row_stride`` pinned bytes (followers of
        a shared pool block here until the leader has created it)."""
        from . import _native

        if self.ptr is not None:
            raise RuntimeError("host pool already allocated")
        if row_stride % 2:
            raise ValueError("row stride must be even")
        self.row_stride = int(row_stride)
        self.nbytes = self.rows * self.row_stride
        if self._share:
            from .replicas import SharedHostPool

            self._shared = SharedHostPool(self._share, self.rows, self.row_stride // 2, leader=self.writable,
                                          publish=False)
            self.ptr = self._shared.ptr
            self.array = self._shared.array
        else:
            host = C.c_void_p()
            dev = C.c_void_p()
            _native.check(
                "spmoe_host_alloc_mapped",
                self._lib.spmoe_host_alloc_mapped(self.nbytes, C.byref(host), C.byref(dev)),
            )
            self.ptr = host.value
            buf = (C.c_uint16 * (self.rows * (self.row_stride // 2))).from_address(self.ptr)
            self.array = np.ctypeslib.as_array(buf).reshape(self.rows, self.row_stride // 2)
        self.tensor = torch.from_numpy(self.array.view(np.int16)).view(torch.bfloat16)
        self.bytes = torch.from_numpy(self.array.view(np.uint8))

    def publish(self) -> None:
        """Leader: mark a shared pool complete (followers unblock)."""
        if self._shared is not None and self.writable:
            self._shared.publish()

    def row_of(self, layer: int, expert: int) -> int:
        return self.index[layer * self.arch.num_experts + expert]

    def blob(self, layer: int, expert: int) -> torch.Tensor:
        """Raw pool row (bf16 expert blob; XC bytes viewed as bf16 with a codec)."""
        return self.tensor[self.row_of(layer, expert)]

    def row_bytes(self, row: int) -> np.ndarray:
        """The bytes of ``row`` that cross the host link (uint8 view)."""
        return self.array[row].view(np.uint8)[: self.wire[row]]

    def raw_row(self, row: int, device=None) -> np.ndarray:
        """Decoded bf16 bits (uint16) of ``row``: the row itself for a raw
        pool, the GPU decoder's output for an XC pool."""
        if self.codec is None:
            return self.array[row]
        from . import codec as X

        hdr = X.header_at(self.ptr + row * self.row_stride)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        blob = self.bytes[row, : int(hdr.blob_bytes)].to(dev)
        out = X.decode(blob, hdr)
        return out.view(torch.int16).cpu().numpy().view(np.uint16)

    def close(self) -> None:
        if getattr(self, "ptr", None):
            self.tensor = None
            self.array = None
            self.bytes = None
            if self._shared is not None:
                self._shared.close(unlink=self.writable)
            else:
                self._lib.spmoe_host_free(C.c_void_p(self.ptr))
            self.ptr = None


# ---------------------------------------------------------------------------
# device weights
# ---------------------------------------------------------------------------
@dataclass
class LayerWeights:
    attn_norm: torch.Tensor
    wqkv: torch.Tensor
    wo: torch.Tensor
    ffn_norm: torch.Tensor
    router: torch.Tensor
    shared: torch.Tensor | None  # [1, 3*Fs*H] blob
    shared_gate: torch.Tensor | None  # [H]
    draft_ffn: torch.Tensor  # [1, 3*Fd*H] blob


@dataclass
class ModelWeights:
    arch: ArchSpec
    embed: torch.Tensor
    layers: list[LayerWeights]
    final_norm: torch.Tensor
    lm_head: torch.Tensor
    rope_cos: torch.Tensor
    rope_sin: torch.Tensor


def _fill(t: torch.Tensor, seed: int, std: float) -> torch.Tensor:
    from .kernels import fill_normal_

    return fill_normal_(t, seed, 0, std)


def build_weights(
    arch: ArchSpec,
    seed: int,
    device: torch.device,
    host_pool: HostExpertPool | None,
    draft_perturb: float = 0.0,
    chunk_experts: int = 8,
) -> ModelWeights:
    """Generate every tensor on the GPU with the counter-hash init; routed
    experts stream to ``host_pool`` (if given) in chunks while their fp32 mean
    accumulates into the draft FFN."""
    H, E, F = arch.hidden, arch.num_experts, arch.ffn
    bf = torch.bfloat16
    std = arch.init_std
    embed = _fill(torch.empty((arch.vocab, H), dtype=bf, device=device), tensor_seed(seed, K_EMBED), arch.embed_std)
    lm_head = _fill(torch.empty((arch.vocab, H), dtype=bf, device=device), tensor_seed(seed, K_LMHEAD), std)
    layers = []
    stage = torch.empty((min(chunk_experts, E), arch.expert_elems), dtype=bf, device=device)
    base_cache: dict[int, torch.Tensor] = {}

    def gen_expert(dst: torch.Tensor, row: int) -> None:
        # expert content is a pure function of its host-pool row, so an
        # aliased row means the same weights for every layer using it
        nonlocal base_cache
        fill_expert_blob(dst, arch, seed, row)
        if arch.expert_spread is not None:
            # upcycled experts: the home layer's shared component plus a
            # per-expert deviation of relative size expert_spread
            base = base_cache.get(row // E)
            if base is None:
                base = torch.empty((arch.expert_elems,), dtype=bf, device=device)
                fill_blob_generic(base, F, H, tensor_seed(seed, K_BASE, row // E), std,
                                  arch.expert_out_scale * arch.res_scale)
                base_cache = {row // E: base}
            dst.copy_((base.float() + dst.float() * arch.expert_spread).to(bf))

    enc = None
    if host_pool is not None and host_pool.codec == "xc":
        from .codec import XcEncoder, expert_segments

        enc = XcEncoder(expert_segments(F, H), device)
        if host_pool.ptr is None:
            # pass 1: every distinct row's blob size -> the pool's row stride
            # (deterministic, so every replica derives the same stride)
            biggest = 0
            for row in range(host_pool.rows):
                gen_expert(stage[0], row)
                hdr = enc.plan(stage[0])
                host_pool.wire[row] = int(hdr.blob_bytes)
                biggest = max(biggest, int(hdr.blob_bytes))
            host_pool.allocate((biggest + 4095) // 4096 * 4096)
            base_cache = {}
    written: set[int] = set()
    for l in range(arch.num_layers):
        wqkv = _fill(torch.empty((arch.qkv_dim, H), dtype=bf, device=device), tensor_seed(seed, K_QKV, l), std)
        wo = _fill(
            torch.empty((H, arch.num_heads * arch.head_dim), dtype=bf, device=device),
            tensor_seed(seed, K_WO, l),
            std * arch.res_scale,
        )
        router = _fill(torch.empty((E, H), dtype=bf, device=device), tensor_seed(seed, K_ROUTER, l), 1.0 / math.sqrt(H))
        acc = torch.zeros((arch.expert_elems,), dtype=torch.float32, device=device)
        for e0 in range(0, E, stage.shape[0]):
            n = min(stage.shape[0], E - e0)
            rows = []
            for j in range(n):
                row = host_pool.row_of(l, e0 + j) if host_pool is not None else l * E + e0 + j
                rows.append(row)
                gen_expert(stage[j], row)
                acc += stage[j].float()
            if host_pool is not None and host_pool.writable:
                for j, row in enumerate(rows):
                    if row in written:
                        continue
                    if enc is None:
                        host_pool.tensor[row].copy_(stage[j], non_blocking=False)
                    else:
                        hdr = enc.plan(stage[j])
                        blob = enc.encode(stage[j], hdr)
                        host_pool.wire[row] = blob.numel()
                        host_pool.bytes[row, : blob.numel()].copy_(blob, non_blocking=False)
                    written.add(row)
        mean = (acc / E).to(bf)
        del acc
        shared = None
        sgate = None
        if arch.shared_ffn:
            shared = torch.empty((1, 3 * arch.shared_ffn * H), dtype=bf, device=device)
            fill_blob_generic(shared[0], arch.shared_ffn, H, tensor_seed(seed, K_SHARED, l), std, arch.expert_out_scale * arch.res_scale)
            if arch.shared_gate:
                sgate = _fill(torch.empty((H,), dtype=bf, device=device), tensor_seed(seed, K_SGATE, l), 1.0 / math.sqrt(H))
        if arch.draft_ffn:
            draft = torch.empty((1, 3 * arch.d_ffn * H), dtype=bf, device=device)
            fill_blob_generic(draft[0], arch.d_ffn, H, tensor_seed(seed, K_EXPERT, l, 10_000), std, arch.expert_out_scale * arch.res_scale)
        else:
            draft = _draft_proxy(arch, mean, shared, router)
        if draft_perturb > 0.0:
            noise = torch.empty_like(draft)
            _fill(noise, tensor_seed(seed, K_PERTURB, l), std * draft_perturb)
            draft = (draft.float() + noise.float()).to(bf)
        layers.append(
            LayerWeights(
                attn_norm=torch.ones((H,), dtype=bf, device=device),
                wqkv=wqkv,
                wo=wo,
                ffn_norm=torch.ones((H,), dtype=bf, device=device),
                router=router,
                shared=shared,
                shared_gate=sgate,
                draft_ffn=draft,
            )
        )
    del stage
    if host_pool is not None:
        torch.cuda.synchronize(device)
        host_pool.publish()
    cos, sin = rope_tables(arch, device)
    return ModelWeights(
        arch=arch,
        embed=embed,
        layers=layers,
        final_norm=torch.ones((H,), dtype=bf, device=device),
        lm_head=lm_head,
        rope_cos=cos,
        rope_sin=sin,
    )


def gate_mass(router: np.ndarray, top_k: int, renorm: bool) -> float:
    """Expected routed gate mass of a router ``[E, H]``: 1 with top-k
    renormalisation, else E[sum of the top-k softmax probabilities] over 512
    seeded N(0, 1) inputs -- host float64 (numpy), so the CPU reference arm
    (oracle/cpu_model.py) derives the identical draft FFN."""
    if renorm:
        return 1.0
    xs = np.random.default_rng(0).standard_normal((512, router.shape[1]))
    lg = xs @ router.astype(np.float64).T
    p = np.exp(lg - lg.max(-1, keepdims=True))
    p /= p.sum(-1, keepdims=True)
    return float(np.sort(p, axis=-1)[:, -top_k:].sum(-1).mean())


def _draft_proxy(arch: ArchSpec, mean: torch.Tensor, shared: torch.Tensor | None, router: torch.Tensor) -> torch.Tensor:
    """Dense draft FFN approximating the layer's MoE: the mean routed expert
    with W2 scaled by the expected routed gate mass (1 with top-k renorm,
    E[sum of the top-k softmax] otherwise, estimated on the router with unit
    RMS inputs), concatenated along F with the shared expert (W2 scaled by
    the expected sigmoid gate, 0.5, for Qwen)."""
    H, F = arch.hidden, arch.ffn
    mass = gate_mass(router.float().cpu().numpy(), arch.top_k, arch.renorm)
    w1 = mean[: F * H].view(F, H)
    w3 = mean[F * H : 2 * F * H].view(F, H)
    w2 = (mean[2 * F * H :].view(H, F).float() * mass).to(mean.dtype)
    if shared is None or arch.shared_gate:
        # a sigmoid-gated shared expert (Qwen1.5-MoE) cannot be folded into
        # one dense FFN (its gate is per token): the draft applies the
        # target's shared expert and gate itself (engine._draft_ffn)
        return torch.cat([w1.reshape(-1), w3.reshape(-1), w2.reshape(-1)]).view(1, -1)
    Fs = arch.shared_ffn
    s = shared[0]
    s1 = s[: Fs * H].view(Fs, H)
    s3 = s[Fs * H : 2 * Fs * H].view(Fs, H)
    s2 = s[2 * Fs * H :].view(H, Fs)
    d1 = torch.cat([w1, s1], dim=0)
    d3 = torch.cat([w3, s3], dim=0)
    d2 = torch.cat([w2, s2], dim=1)
    return torch.cat([d1.reshape(-1), d3.reshape(-1), d2.reshape(-1)]).view(1, -1)


def fill_blob_generic(blob: torch.Tensor, F: int, H: int, seed: int, std: float, out_scale: float) -> None:
    """W1|W3 ~ N(0, std^2), W2 ~ N(0, (std*out_scale)^2), each with its own
    counter stream (offset 0 of three sub-seeds)."""
    n13 = F * H
    _fill(blob[:n13], _splitmix64(seed ^ 1), std)
    _fill(blob[n13 : 2 * n13], _splitmix64(seed ^ 3), std)
    _fill(blob[2 * n13 : 3 * n13], _splitmix64(seed ^ 2), std * out_scale)


def fill_expert_blob(blob: torch.Tensor, arch: ArchSpec, seed: int, row: int) -> None:
    """Routed expert content is a function of its host-pool row (row =
    layer*E + expert unless the pool aliases)."""
    fill_blob_generic(
        blob, arch.ffn, arch.hidden, tensor_seed(seed, K_EXPERT, row), arch.init_std, arch.expert_out_scale * arch.res_scale
    )


# ---------------------------------------------------------------------------
# transformer pieces (torch; off the hot path)
# ---------------------------------------------------------------------------
def rope_tables_host(arch: ArchSpec) -> tuple[np.ndarray, np.ndarray]:
    """Rotate-half RoPE tables ``[max_seq, head_dim]`` f32, computed on the
    host with libm (``math``: correctly rounded double cos/sin, independent
    of the CPU's SIMD extensions) so the device and the CPU oracle use the
    same bits.  inv_freq_i = 1 / theta^(2i/d); angle = pos * inv_freq."""
    d = arch.head_dim
    inv = [1.0 / (arch.rope_theta ** (i / d)) for i in range(0, d, 2)]
    cos = np.empty((arch.max_seq, d), np.float32)
    sin = np.empty((arch.max_seq, d), np.float32)
    for p in range(arch.max_seq):
        c = [math.cos(p * f) for f in inv]
        s_ = [math.sin(p * f) for f in inv]
        cos[p] = c + c
        sin[p] = s_ + s_
    return cos, sin


def rope_tables(arch: ArchSpec, device) -> tuple[torch.Tensor, torch.Tensor]:
    cos, sin = rope_tables_host(arch)
    return torch.from_numpy(cos).to(device), torch.from_numpy(sin).to(device)


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """bf16 RMSNorm (csrc/spmoe_attn.cu; fixed-order fp32 math, IEEE sqrt/div)."""
    from .kernels import rms_norm as _rms

    return _rms(x, w, eps, out=out)


class KVCache:
    """Per-model KV cache ``[L, B, n_kv, S, hd]`` (keys of one head contiguous
    for the attention kernel); positions are per-sequence lengths."""

    def __init__(self, arch: ArchSpec, batch: int, device, max_seq: int | None = None):
        S = max_seq or arch.max_seq
        shape = (arch.num_layers, batch, arch.num_kv_heads, S, arch.head_dim)
        self.k = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.v = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.max_seq = S


def attention_block(
    w: ModelWeights,
    layer: int,
    x: torch.Tensor,  # [B, T, H] residual stream
    kv: KVCache,
    start: torch.Tensor,  # [B] int64 position of the first of the T tokens
    out: torch.Tensor | None = None,
) -> torch.Tensor:
    """The attention half of a decoder layer: RMSNorm fused into the qkv
    projection (K9) -> RoPE + KV append -> causal GQA attention over the
    cache -> W_o projection fused with the residual add (K9):
    ``bf16(x + bf16(attn(norm(x)) W_o^T))``; ``out=x`` updates in place."""
    from . import kernels as K

    a = w.arch
    lw = w.layers[layer]
    qkv = K.linear(x, lw.wqkv, norm_w=lw.attn_norm, eps=a.rms_eps)
    q = K.rope_kv(qkv, w.rope_cos, w.rope_sin, start, a.num_heads, a.num_kv_heads, a.head_dim, kv.k[layer],
                  kv.v[layer])
    o = K.attention_cached(q, kv.k[layer], kv.v[layer], start)
    return K.linear(o, lw.wo, residual=x, out=out)


def lm_logits(w: ModelWeights, x: torch.Tensor) -> torch.Tensor:
    """Final RMSNorm fused into the lm_head projection, fp32 logits."""
    from . import kernels as K

    return K.linear(x, w.lm_head, norm_w=w.final_norm, eps=w.arch.rms_eps, f32=True)
