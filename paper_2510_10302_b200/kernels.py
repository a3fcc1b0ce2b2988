"""Torch-tensor front end of the sm_100a kernels (K1-K6 of SURVEY.md §2.1).

Thin: validates dtypes/shapes/devices, passes raw pointers and the current
CUDA stream to the C ABI (:mod:`._native`), returns torch tensors.  No
computation happens here and there is no fallback path.
"""

from __future__ import annotations

from typing import Sequence

import torch

from . import _native

# launches of spmoe kernels issued through this module (bench.py reports the
# count inside its timed region as ``gpu_launches``)
LAUNCHES = {"count": 0}

BF16 = torch.bfloat16
F32 = torch.float32
I32 = torch.int32


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype, name: str, ndim: int | None = None) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dims, got {t.dim()}")


# ---------------------------------------------------------------------------
# K1
# ---------------------------------------------------------------------------
def router_topk(
    x: torch.Tensor,
    w_gate: torch.Tensor,
    k: int,
    renorm: bool = True,
    *,
    want_logits: bool = False,
    host_idx_dev_ptr: int | None = None,
    shared_gate_w: torch.Tensor | None = None,
    out: tuple[torch.Tensor, torch.Tensor] | None = None,
    logits_out: torch.Tensor | None = None,
    stream=None,
):
    """Fused router projection + top-k + softmax weights.

    Returns ``(weights f32[T,k], idx i32[T,k], logits f32[T,E] | None,
    shared_gate f32[T] | None)``.
    """
    _need(x, BF16, "x", 2)
    _need(w_gate, BF16, "w_gate", 2)
    T, H = x.shape
    E = w_gate.shape[0]
    if w_gate.shape[1] != H:
        raise ValueError("router weight hidden size mismatch")
    if out is None:
        weights = torch.empty((T, k), dtype=F32, device=x.device)
        idx = torch.empty((T, k), dtype=I32, device=x.device)
    else:
        weights, idx = out
    logits = logits_out if logits_out is not None else (
        torch.empty((T, E), dtype=F32, device=x.device) if want_logits else None)
    sg = None
    if shared_gate_w is not None:
        _need(shared_gate_w, BF16, "shared_gate_w")
        sg = torch.empty((T,), dtype=F32, device=x.device)
    LAUNCHES["count"] += 1
    _native.call(
        "spmoe_router_topk",
        x.data_ptr(),
        w_gate.data_ptr(),
        T,
        H,
        E,
        k,
        1 if renorm else 0,
        weights.data_ptr(),
        idx.data_ptr(),
        _ptr(logits),
        host_idx_dev_ptr,
        _ptr(shared_gate_w),
        _ptr(sg),
        _stream(stream),
    )
    return weights, idx, logits, sg


# ---------------------------------------------------------------------------
# K2
# ---------------------------------------------------------------------------
def moe_permute(idx: torch.Tensor, num_experts: int, out=None, stream=None):
    """Group routed (token, choice) pairs by expert, stable by token."""
    _need(idx, I32, "idx", 2)
    T, k = idx.shape
    if out is None:
        offsets = torch.empty((num_experts + 1,), dtype=I32, device=idx.device)
        perm = torch.empty((T * k,), dtype=I32, device=idx.device)
        inv = torch.empty((T * k,), dtype=I32, device=idx.device)
    else:
        offsets, perm, inv = out
    LAUNCHES["count"] += 1
    _native.call(
        "spmoe_moe_permute",
        idx.data_ptr(),
        T,
        k,
        num_experts,
        offsets.data_ptr(),
        perm.data_ptr(),
        inv.data_ptr(),
        _stream(stream),
    )
    return offsets, perm, inv


# ---------------------------------------------------------------------------
# K3
# ---------------------------------------------------------------------------
def _slot_array(slots: Sequence[int], E: int):
    import ctypes

    arr = (ctypes.c_int32 * max(E, 1))()
    for e in range(E):
        arr[e] = int(slots[e]) if slots[e] is not None and slots[e] >= 0 else 0
    return arr


def expert_ffn(
    pool: torch.Tensor,
    slot_of_expert: Sequence[int],
    expert_mask: int,
    x: torch.Tensor,
    ffn_dim: int,
    top_k: int,
    offsets: torch.Tensor,
    perm: torch.Tensor,
    h_scratch: torch.Tensor,
    y: torch.Tensor,
    max_tokens_per_expert: int = 0,
    phase: str = "both",
    stream=None,
) -> None:
    """Grouped SwiGLU of the experts in ``expert_mask`` reading the slot pool.

    ``pool`` is ``[S, 3*F*H]`` bf16 (one expert blob per slot); ``y`` receives
    ``[T*k, H]`` fp32 rows in permuted order.
    """
    _need(pool, BF16, "pool", 2)
    _need(x, BF16, "x", 2)
    T, H = x.shape
    E = len(slot_of_expert)
    slot_elems = pool.shape[1]
    if slot_elems < 3 * ffn_dim * H:
        raise ValueError("slot too small for the expert blob")
    slots = _slot_array(slot_of_expert, E)
    st = _stream(stream)
    if phase == "both":
        LAUNCHES["count"] += 2
        _native.call(
            "spmoe_expert_ffn", pool.data_ptr(), slot_elems, slots, expert_mask, x.data_ptr(), T, H, ffn_dim, E,
            top_k, offsets.data_ptr(), perm.data_ptr(), h_scratch.data_ptr(), y.data_ptr(),
            max_tokens_per_expert, st,
        )
        return
    if phase == "up":
        LAUNCHES["count"] += 1
        _native.call(
            "spmoe_expert_ffn_up",
            pool.data_ptr(),
            slot_elems,
            slots,
            expert_mask,
            x.data_ptr(),
            T,
            H,
            ffn_dim,
            E,
            top_k,
            offsets.data_ptr(),
            perm.data_ptr(),
            h_scratch.data_ptr(),
            max_tokens_per_expert,
            st,
        )
    if phase == "down":
        LAUNCHES["count"] += 1
        _native.call(
            "spmoe_expert_ffn_down",
            pool.data_ptr(),
            slot_elems,
            slots,
            expert_mask,
            T,
            H,
            ffn_dim,
            E,
            top_k,
            offsets.data_ptr(),
            h_scratch.data_ptr(),
            y.data_ptr(),
            max_tokens_per_expert,
            st,
        )


def tc_split(ffn_dim: int) -> int:
    """Upper bound of the split-K factor for a reduction of ``ffn_dim``
    (sizes the workspace): at most 16, at least 4 K-blocks of 64 per split."""
    kb = ffn_dim // 64
    return max(1, min(16, kb // 4))


def tc_plan(token_counts, hidden: int, ffn_dim: int, sms: int = 148) -> tuple[int, int]:
    """(split_up, split_dn) for the tcgen05 K3 launch of experts with the
    given routed-token counts.

    Rule measured on B200 (tools/tc_split_sweep.py, profiles/r1_tc_split_sweep.jsonl):
    splitting never pays when the phase already has >= ~0.85 x SMs tiles
    (the fixed-order partial reduction costs more than the tail it removes),
    and the up phase always has enough (F/128 = 112 tiles per Mixtral
    expert).  The down phase of one or two experts (32 tiles each) does not:
    split K so that tiles x split reaches ~0.85 x SMs (1 expert: 3.3 -> 4.3
    TB/s, 2 experts: 4.6 -> 5.1 TB/s)."""
    chunks = sum((int(c) + 63) // 64 for c in token_counts if c > 0)
    if chunks == 0:
        return 1, 1
    tiles_dn = chunks * (hidden // 128)
    want = 0.85 * sms
    sd = 1 if tiles_dn >= want else -(-int(want) // tiles_dn)
    sd = max(1, min(sd, 16, (ffn_dim // 64) // 4))
    return 1, sd


def tc_plan_static(hidden: int, ffn_dim: int, sms: int = 148) -> tuple[int, int]:
    """Launch-independent (split_up, split_dn): the split a lone 1-token
    expert would get, capped at one split per 1024 of ``ffn_dim`` (short
    reductions never pay, sweep rows deepseek_*/qwen_*).  Because it does not
    depend on which experts share a launch, every expert's output bits are the
    same whether it runs in the cached-first group or alone after its copy
    lands -- the engine's tokens are reproducible run to run.  Cost vs the
    per-launch plan on the Mixtral sweep: <= 1.7 % (T=72), 0.3 % (T=5)."""
    _, sd = tc_plan([1], hidden, ffn_dim, sms)
    return 1, max(1, min(sd, ffn_dim // 1024))


def tc_workspace_floats(rows: int, hidden: int, ffn_dim: int, split_up: int, split_dn: int) -> int:
    return max(2 * split_up * rows * ffn_dim if split_up > 1 else 0, split_dn * rows * hidden if split_dn > 1 else 0)


def expert_ffn_tc(
    pool: torch.Tensor,
    slot_of_expert: Sequence[int],
    expert_mask: int,
    x: torch.Tensor,
    ffn_dim: int,
    top_k: int,
    offsets: torch.Tensor,
    perm: torch.Tensor,
    x_perm: torch.Tensor,
    h_scratch: torch.Tensor,
    y: torch.Tensor,
    workspace: torch.Tensor | None,
    split_up: int = 1,
    split_dn: int = 1,
    stream=None,
) -> None:
    """tcgen05/TMEM/TMA grouped SwiGLU (same outputs as :func:`expert_ffn`);
    ``workspace`` f32 of :func:`tc_workspace_floats` elements holds the
    split-K partials (see :func:`tc_plan`)."""
    _need(pool, BF16, "pool", 2)
    _need(x, BF16, "x", 2)
    T, H = x.shape
    E = len(slot_of_expert)
    if split_up > 1 or split_dn > 1:
        need = tc_workspace_floats(T * top_k, H, ffn_dim, split_up, split_dn)
        if workspace is None or workspace.numel() < need:
            raise ValueError(f"tcgen05 workspace needs {need} floats")
    LAUNCHES["count"] += 3 + (split_up > 1) + (split_dn > 1)
    _native.call(
        "spmoe_expert_ffn_tc",
        pool.data_ptr(),
        pool.shape[1],
        _slot_array(slot_of_expert, E),
        expert_mask,
        x.data_ptr(),
        T,
        H,
        ffn_dim,
        E,
        top_k,
        offsets.data_ptr(),
        perm.data_ptr(),
        x_perm.data_ptr(),
        h_scratch.data_ptr(),
        y.data_ptr(),
        _ptr(workspace),
        split_up,
        split_dn,
        _stream(stream),
    )


def expert_ffn_tc_fused(
    pool: torch.Tensor,
    slot_of_expert: Sequence[int],
    expert_mask: int,
    x: torch.Tensor,
    ffn_dim: int,
    top_k: int,
    offsets: torch.Tensor,
    perm: torch.Tensor,
    x_perm: torch.Tensor,
    h_scratch: torch.Tensor,
    y: torch.Tensor,
    workspace: torch.Tensor | None,
    split_dn: int,
    grid_sync: torch.Tensor,
    stream=None,
) -> None:
    """Single cooperative launch of both tcgen05 phases (grid barrier between
    them); ``grid_sync`` is a 1-element int32 device tensor."""
    _need(pool, BF16, "pool", 2)
    _need(x, BF16, "x", 2)
    T, H = x.shape
    E = len(slot_of_expert)
    if split_dn > 1:
        need = split_dn * T * top_k * H
        if workspace is None or workspace.numel() < need:
            raise ValueError(f"tcgen05 workspace needs {need} floats")
    LAUNCHES["count"] += 2 + (split_dn > 1)
    _native.call(
        "spmoe_expert_ffn_tc_fused",
        pool.data_ptr(),
        pool.shape[1],
        _slot_array(slot_of_expert, E),
        expert_mask,
        x.data_ptr(),
        T,
        H,
        ffn_dim,
        E,
        top_k,
        offsets.data_ptr(),
        perm.data_ptr(),
        x_perm.data_ptr(),
        h_scratch.data_ptr(),
        y.data_ptr(),
        _ptr(workspace),
        split_dn,
        grid_sync.data_ptr(),
        _stream(stream),
    )


UNIT_MAX_TOKENS = 16


def tc_units_workspace_floats(rows: int, hidden: int, ffn_dim: int) -> int:
    return (ffn_dim // 128) * rows * hidden


def expert_ffn_tc_units(
    pool: torch.Tensor,
    slot_of_expert: Sequence[int],
    expert_mask: int,
    x: torch.Tensor,
    ffn_dim: int,
    top_k: int,
    offsets: torch.Tensor,
    perm: torch.Tensor,
    max_tokens_per_expert: int,
    x_perm: torch.Tensor | None,
    h_scratch: torch.Tensor | None,
    y: torch.Tensor,
    workspace: torch.Tensor,
    stream=None,
) -> None:
    """Unit-fused tcgen05 K3: one launch runs both phases per (expert,
    128-feature block) unit, a PDL-chained one sums the partials in a fixed
    order; experts with at most :data:`UNIT_MAX_TOKENS` routed tokens.
    ``workspace``: f32 of :func:`tc_units_workspace_floats` elements.
    ``x_perm`` is unused (the kernel gathers x rows itself by TMA gather4)
    and may be None."""
    _need(pool, BF16, "pool", 2)
    _need(x, BF16, "x", 2)
    T, H = x.shape
    E = len(slot_of_expert)
    if max_tokens_per_expert > UNIT_MAX_TOKENS:
        raise ValueError(f"expert_ffn_tc_units takes <= {UNIT_MAX_TOKENS} tokens per expert")
    need = tc_units_workspace_floats(T * top_k, H, ffn_dim)
    if workspace is None or workspace.numel() < need:
        raise ValueError(f"tcgen05 unit workspace needs {need} floats")
    LAUNCHES["count"] += 2  # unit kernel (x rows by TMA gather4) + fixed-order reduce
    _native.call(
        "spmoe_expert_ffn_tc_units",
        pool.data_ptr(),
        pool.shape[1],
        _slot_array(slot_of_expert, E),
        expert_mask,
        x.data_ptr(),
        T,
        H,
        ffn_dim,
        E,
        top_k,
        offsets.data_ptr(),
        perm.data_ptr(),
        max_tokens_per_expert,
        _ptr(x_perm),
        _ptr(h_scratch),
        y.data_ptr(),
        workspace.data_ptr(),
        _stream(stream),
    )


# ---------------------------------------------------------------------------
# K4
# ---------------------------------------------------------------------------
def moe_combine(
    y: torch.Tensor | None,
    inv_pos: torch.Tensor | None,
    weights: torch.Tensor | None,
    T: int,
    H: int,
    k: int,
    *,
    residual: torch.Tensor | None = None,
    y_shared: torch.Tensor | None = None,
    shared_gate: torch.Tensor | None = None,
    out: torch.Tensor | None = None,
    device=None,
    stream=None,
) -> torch.Tensor:
    dev = device or (y.device if y is not None else residual.device)
    if out is None:
        out = torch.empty((T, H), dtype=BF16, device=dev)
    LAUNCHES["count"] += 1
    _native.call(
        "spmoe_moe_combine",
        _ptr(y),
        _ptr(inv_pos),
        _ptr(weights),
        T,
        H,
        k,
        _ptr(y_shared),
        _ptr(shared_gate),
        _ptr(residual),
        out.data_ptr(),
        _stream(stream),
    )
    return out


# ---------------------------------------------------------------------------
# layer block around the MoE (csrc/spmoe_attn.cu)
# ---------------------------------------------------------------------------
def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float, out: torch.Tensor | None = None, stream=None):
    """bf16 RMSNorm over the last dim (fp32 math, one rounding)."""
    _need(w, BF16, "w", 1)
    if x.dtype != BF16 or not x.is_cuda:
        raise ValueError("x must be a CUDA bf16 tensor (no CPU fallback)")
    x = x.contiguous()
    H = x.shape[-1]
    if out is None:
        out = torch.empty_like(x)
    LAUNCHES["count"] += 1
    _native.call("spmoe_rms_norm", x.data_ptr(), w.data_ptr(), x.numel() // H, H, float(eps), out.data_ptr(),
                 _stream(stream))
    return out


def rope_kv(qkv: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, start: torch.Tensor, nh: int, nkv: int,
            hd: int, k_cache: torch.Tensor, v_cache: torch.Tensor, stream=None) -> torch.Tensor:
    """qkv ``[B, T, (nh+2nkv)*hd]`` -> rotated q ``[B, nh, T, hd]``; rotated k
    and v appended to the layer caches ``[B, nkv, S, hd]`` at start[b]+t."""
    B, T = qkv.shape[0], qkv.shape[1]
    qkv = qkv.contiguous()
    if start.dtype != torch.int64 or not start.is_cuda:
        raise ValueError("start must be a CUDA int64 tensor")
    q = torch.empty((B, nh, T, hd), dtype=BF16, device=qkv.device)
    LAUNCHES["count"] += 1
    _native.call("spmoe_rope_kv", qkv.data_ptr(), cos.data_ptr(), sin.data_ptr(), start.data_ptr(), B, T, nh, nkv,
                 hd, k_cache.shape[2], cos.shape[0], q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(),
                 _stream(stream))
    return q


def linear(x: torch.Tensor, w: torch.Tensor, *, norm_w: torch.Tensor | None = None, eps: float = 0.0,
           out_f32: torch.Tensor | None = None, out: torch.Tensor | None = None,
           residual: torch.Tensor | None = None, f32: bool = False, stream=None) -> torch.Tensor:
    """K9: ``x [..., K] @ w[N, K]^T`` with the fixed-order dot product.

    ``norm_w``: RMSNorm x first (fused).  ``f32`` / ``out_f32``: fp32 output
    (logits); else bf16, or ``bf16(residual + bf16(y))`` with ``residual``
    (``out`` may be ``residual`` itself: in place)."""
    _need(w, BF16, "w", 2)
    if x.dtype != BF16 or not x.is_cuda:
        raise ValueError("x must be a CUDA bf16 tensor (no CPU fallback)")
    N, K = w.shape
    if x.shape[-1] != K:
        raise ValueError("linear: x and w disagree on K")
    x2 = x.reshape(-1, K)
    if x2.stride(-1) != 1:
        x2 = x2.contiguous()
    T = x2.shape[0]
    lead = tuple(x.shape[:-1])
    y32 = yb = None
    if f32 or out_f32 is not None:
        y32 = out_f32 if out_f32 is not None else torch.empty(lead + (N,), dtype=F32, device=x.device)
        res = y32
    else:
        yb = out if out is not None else torch.empty(lead + (N,), dtype=BF16, device=x.device)
        res = yb
    if residual is not None:
        _need(residual, BF16, "residual")
        if residual.numel() != T * N:
            raise ValueError("residual shape mismatch")
    if norm_w is not None:
        _need(norm_w, BF16, "norm_w", 1)
    LAUNCHES["count"] += 1
    _native.call("spmoe_linear", w.data_ptr(), x2.data_ptr(), x2.stride(0), T, K, N, _ptr(norm_w), float(eps),
                 _ptr(y32), N if y32 is not None else 0, _ptr(yb), _ptr(residual), _stream(stream))
    return res


def attention_cached(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, start: torch.Tensor,
                     stream=None) -> torch.Tensor:
    """Causal GQA attention of q ``[B, nh, T, hd]`` over the caches; returns
    ``[B, T, nh*hd]`` bf16."""
    B, nh, T, hd = q.shape
    nkv, S = k_cache.shape[1], k_cache.shape[2]
    out = torch.empty((B, T, nh * hd), dtype=BF16, device=q.device)
    LAUNCHES["count"] += 1
    _native.call("spmoe_attention", q.data_ptr(), k_cache.data_ptr(), v_cache.data_ptr(), start.data_ptr(), B, T,
                 nh, nkv, hd, S, float(hd ** -0.5), out.data_ptr(), _stream(stream))
    return out


def gather_rows(src: torch.Tensor, idx: torch.Tensor, div: int = 1, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """``out[j] = src[idx[j] // div]`` (rows of any dtype, row bytes a
    multiple of 4): packs / unpacks the expert-parallel exchange buffers."""
    if not src.is_cuda or not src.is_contiguous():
        raise ValueError("src must be a contiguous CUDA tensor (no CPU fallback)")
    _need(idx, I32, "idx", 1)
    n = idx.shape[0]
    if out is None:
        out = torch.empty((n,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    if n == 0:
        return out
    row_bytes = (src.numel() // max(src.shape[0], 1)) * src.element_size()
    LAUNCHES["count"] += 1
    _native.call("spmoe_gather_rows", src.data_ptr(), idx.data_ptr(), n, div, row_bytes, out.data_ptr(),
                 _stream(stream))
    return out


# ---------------------------------------------------------------------------
# K6
# ---------------------------------------------------------------------------
def greedy_accept(logits: torch.Tensor, draft: torch.Tensor, stream=None):
    """logits f32 [B, N+1, V]; draft i32 [B, N] -> (argmax [B,N+1], result [B,2])."""
    _need(logits, F32, "logits", 3)
    B, N1, V = logits.shape
    N = N1 - 1
    if N > 0:
        _need(draft, I32, "draft", 2)
    amax = torch.empty((B, N1), dtype=I32, device=logits.device)
    res = torch.empty((B, 2), dtype=I32, device=logits.device)
    LAUNCHES["count"] += 2
    _native.call(
        "spmoe_greedy_accept",
        logits.data_ptr(),
        V,
        draft.data_ptr() if N > 0 else None,
        B,
        N,
        V,
        amax.data_ptr(),
        res.data_ptr(),
        _stream(stream),
    )
    return amax, res


def argmax_rows(logits: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    _need(logits, F32, "logits", 2)
    R, V = logits.shape
    if out is None:
        out = torch.empty((R,), dtype=I32, device=logits.device)
    LAUNCHES["count"] += 1
    _native.call("spmoe_argmax_rows", logits.data_ptr(), V, R, V, out.data_ptr(), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# init
# ---------------------------------------------------------------------------
def fill_normal_(t: torch.Tensor, seed: int, offset: int = 0, std: float = 0.02, stream=None):
    """Deterministic counter-hash N(0, std^2) fill (bit-identical on CPU)."""
    _need(t, BF16, "t")
    _native.call(
        "spmoe_fill_normal_bf16",
        t.data_ptr(),
        t.numel(),
        seed & 0xFFFFFFFFFFFFFFFF,
        offset & 0xFFFFFFFFFFFFFFFF,
        float(std),
        _stream(stream),
    )
    return t
