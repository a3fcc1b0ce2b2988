"""Parity of the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar: bit-exact.  Every kernel follows the fixed-order arithmetic contract of
include/spmoe.h, which oracle/spmoe_oracle.c restates, so routing indices,
softmax weights, router logits, SwiGLU activations, expert outputs, combined
hidden states and accepted tokens must match bit for bit (tolerance 0).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def bits(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return t.contiguous().cpu().numpy()


def _native_lib():
    from paper_2510_10302_b200 import _native

    return _native.load()


def to_dev_bf16(a_u16: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(a_u16.view(np.int16).copy()).view(torch.bfloat16).cuda()


def rand_bf16(shape, seed, std=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(shape, generator=g) * std).to(torch.bfloat16)


def same_bits(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.dtype == np.float32:
        return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))
    return np.array_equal(a, b)


ROUTER_CASES = [
    # (T, H, E, k, renorm, shared_gate)
    (5, 256, 8, 2, True, False),  # tiny
    (5, 4096, 8, 2, True, False),  # Mixtral verify N=4
    (72, 4096, 8, 2, True, False),  # Mixtral batch 8 x N 8
    (1, 4096, 8, 1, True, False),  # predictor, prefetch_k = 1
    (5, 2048, 64, 6, False, False),  # DeepSeek-V2-Lite
    (9, 2048, 60, 4, False, True),  # Qwen1.5-MoE + shared gate
]


@pytest.mark.parametrize("T,H,E,k,renorm,sg", ROUTER_CASES)
def test_router_topk_bit_exact(oracle, T, H, E, k, renorm, sg):
    from paper_2510_10302_b200 import kernels as K

    x = rand_bf16((T, H), 1 + T + H)
    w = rand_bf16((E, H), 2 + E, std=1.0 / np.sqrt(H))
    sgw = rand_bf16((H,), 3, std=1.0 / np.sqrt(H)) if sg else None
    wd, idd, lgd, sgd = K.router_topk(
        x.cuda(), w.cuda(), k, renorm, want_logits=True, shared_gate_w=None if sgw is None else sgw.cuda()
    )
    torch.cuda.synchronize()
    wo, io, lo, so = oracle.router_topk(bits(x), bits(w), k, renorm, None if sgw is None else bits(sgw))
    assert same_bits(bits(lgd), lo)
    assert np.array_equal(bits(idd), io)
    assert same_bits(bits(wd), wo)
    if sg:
        assert same_bits(bits(sgd), so)


def test_router_ties_lowest_index(oracle):
    """Exact logit ties (duplicated router rows) resolve to the lowest index,
    the reference tie-break (trace.py:28-37)."""
    from paper_2510_10302_b200 import kernels as K

    H, E, k, T = 512, 16, 4, 33
    w = rand_bf16((E, H), 9, std=0.05)
    w[5] = w[2]
    w[11] = w[2]
    w[7] = w[3]
    x = rand_bf16((T, H), 10)
    x[0] = 0.0  # all logits tie at 0 -> (0, 1, 2, 3)
    wd, idd, _, _ = K.router_topk(x.cuda(), w.cuda(), k, True)
    torch.cuda.synchronize()
    wo, io, _, _ = oracle.router_topk(bits(x), bits(w), k, True)
    assert np.array_equal(bits(idd), io)
    assert list(bits(idd)[0]) == [0, 1, 2, 3]
    assert same_bits(bits(wd), wo)
    # where row 2 is selected, rows 5 and 11 (equal logits) follow in index order
    for t in range(T):
        sel = list(bits(idd)[t])
        if 5 in sel:
            assert 2 in sel and sel.index(2) < sel.index(5)


def test_router_many_tokens_indices(oracle):
    """>= 10^4 random token vectors: routing indices bit-exact."""
    from paper_2510_10302_b200 import kernels as K

    T, H, E, k = 10240, 256, 8, 2
    x = rand_bf16((T, H), 77)
    w = rand_bf16((E, H), 78, std=1 / 16)
    wd, idd, _, _ = K.router_topk(x.cuda(), w.cuda(), k, True)
    torch.cuda.synchronize()
    wo, io, _, _ = oracle.router_topk(bits(x), bits(w), k, True)
    assert np.array_equal(bits(idd), io)
    assert same_bits(bits(wd), wo)


def test_router_host_mapped_handoff(oracle):
    """K1 writes the indices into mapped pinned memory (Alg. 1 hand-off)."""
    from paper_2510_10302_b200 import kernels as K
    from paper_2510_10302_b200.predictor import DraftGuidedPredictor

    ring = DraftGuidedPredictor(entries=4, width=3)
    try:
        x = rand_bf16((1, 4096), 5)
        w = rand_bf16((64, 4096), 6, std=1 / 64)
        i, hptr, ev = ring.predict(x.cuda(), w.cuda(), 3, False, torch.empty((1, 3), device="cuda"),
                                   torch.empty((1, 3), dtype=torch.int32, device="cuda"))
        _native_lib().spmoe_event_synchronize(ev)
        _, io, _, _ = oracle.router_topk(bits(x), bits(w), 3, False)
        assert list(ring.view[i]) == list(io[0])
    finally:
        ring.close()


@pytest.mark.parametrize("T,k,E", [(5, 2, 8), (72, 2, 8), (9, 6, 64), (1, 1, 8), (17, 4, 60)])
def test_permute_exact(oracle, T, k, E):
    from paper_2510_10302_b200 import kernels as K

    rng = np.random.default_rng(T * 100 + E)
    idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    off, perm, inv = K.moe_permute(torch.from_numpy(idx).cuda(), E)
    torch.cuda.synchronize()
    o2, p2, i2 = oracle.moe_permute(idx, E)
    assert np.array_equal(bits(off), o2)
    assert np.array_equal(bits(perm), p2)
    assert np.array_equal(bits(inv), i2)


def _ffn_case(oracle, T, H, F, E, k, seed, hints=(0,), masks=None):
    from paper_2510_10302_b200 import kernels as K

    rng = np.random.default_rng(seed)
    x = rand_bf16((T, H), seed)
    idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    pool = torch.empty((E + 2, 3 * F * H), dtype=torch.bfloat16, device="cuda")
    K.fill_normal_(pool, seed + 1, 0, 0.02)
    slots = list(rng.permutation(E + 2)[:E])  # experts live in scattered slots
    idx_d = torch.from_numpy(idx).cuda()
    off, perm, inv = K.moe_permute(idx_d, E)
    n = T * k
    pool_h = bits(pool)
    blobs = [pool_h[slots[e]] for e in range(E)]
    o2, p2, _ = oracle.moe_permute(idx, E)
    h_ref, y_ref = oracle.expert_ffn(blobs, bits(x), F, o2, p2)
    xd = x.cuda()
    for hint in hints:
        for mask_list in masks or [[(1 << E) - 1]]:
            h = torch.zeros((n, F), dtype=torch.bfloat16, device="cuda")
            y = torch.zeros((n, H), dtype=torch.float32, device="cuda")
            for m in mask_list:
                K.expert_ffn(pool, slots, m, xd, F, k, off, perm, h, y, hint)
            torch.cuda.synchronize()
            assert same_bits(bits(h), h_ref[:n]), f"h mismatch hint={hint}"
            assert same_bits(bits(y), y_ref[:n]), f"y mismatch hint={hint}"
    return pool, slots, x, idx


def test_expert_ffn_tiny_all_tiles(oracle):
    _ffn_case(oracle, T=5, H=256, F=512, E=8, k=2, seed=3, hints=(0, 1, 2, 4, 8))


def test_expert_ffn_masks_cached_first(oracle):
    """Running resident experts first and late experts one by one (cached-
    first order, §4.3) gives the same bits as one launch."""
    E = 8
    _ffn_case(oracle, T=5, H=256, F=512, E=E, k=2, seed=4,
              masks=[[0b00001111, 1 << 4, 1 << 5, 1 << 6, 1 << 7], [(1 << E) - 1]])


def test_expert_ffn_mixtral_shape(oracle):
    oracle.set_threads(16)
    _ffn_case(oracle, T=5, H=4096, F=14336, E=8, k=2, seed=5, hints=(0, 2))


def test_expert_ffn_deepseek_shape(oracle):
    oracle.set_threads(16)
    _ffn_case(oracle, T=9, H=2048, F=1408, E=64, k=6, seed=6, hints=(0, 1))


def test_expert_ffn_many_tokens_per_expert(oracle):
    # T_e well above the register tile (token-tile loop)
    _ffn_case(oracle, T=40, H=256, F=512, E=4, k=2, seed=8, hints=(0, 4, 8))


def test_combine_exact(oracle):
    from paper_2510_10302_b200 import kernels as K

    T, H, k = 9, 2048, 4
    rng = np.random.default_rng(1)
    y = rng.standard_normal((T * k, H)).astype(np.float32)
    inv = rng.permutation(T * k).astype(np.int32)
    w = rng.random((T, k)).astype(np.float32)
    ys = rng.standard_normal((T, H)).astype(np.float32)
    sg = rng.random(T).astype(np.float32)
    res = bits(rand_bf16((T, H), 2))
    for kwargs in ({}, {"ys": ys}, {"ys": ys, "sg": sg}, {"residual": res}, {"ys": ys, "sg": sg, "residual": res}):
        out = K.moe_combine(
            torch.from_numpy(y).cuda(), torch.from_numpy(inv).cuda(), torch.from_numpy(w).cuda(), T, H, k,
            residual=to_dev_bf16(kwargs["residual"]) if "residual" in kwargs else None,
            y_shared=torch.from_numpy(kwargs["ys"]).cuda() if "ys" in kwargs else None,
            shared_gate=torch.from_numpy(kwargs["sg"]).cuda() if "sg" in kwargs else None,
        )
        torch.cuda.synchronize()
        ref = oracle.moe_combine(y, inv, w, T, H, k, kwargs.get("ys"), kwargs.get("sg"), kwargs.get("residual"))
        assert same_bits(bits(out), ref)


def test_greedy_accept_exact(oracle):
    from paper_2510_10302_b200 import kernels as K

    B, N, V = 8, 4, 32000
    rng = np.random.default_rng(2)
    logits = rng.standard_normal((B, N + 1, V)).astype(np.float32)
    amax_true = logits.argmax(-1)
    draft = amax_true[:, :N].copy().astype(np.int32)
    for b in range(B):  # reject at position b (b >= N: all accepted)
        if b < N:
            draft[b, b] = (draft[b, b] + 1) % V
    top = logits[7, 4].max() + 1.0  # exact tie on the bonus row -> lowest index
    logits[7, 4, 17] = top
    logits[7, 4, 5] = top
    am, res = K.greedy_accept(torch.from_numpy(logits).cuda(), torch.from_numpy(draft).cuda())
    torch.cuda.synchronize()
    am2, res2 = oracle.greedy_accept(logits, draft)
    assert np.array_equal(bits(am), am2)
    assert np.array_equal(bits(res), res2)
    assert am2[7, 4] == 5 and res2[7, 1] == 5 and res2[7, 0] == N
    assert [int(r[0]) for r in res2[:4]] == [0, 1, 2, 3]


def test_fill_normal_matches_oracle(oracle):
    from paper_2510_10302_b200 import kernels as K

    t = torch.empty((1 << 20) + 3, dtype=torch.bfloat16, device="cuda")
    K.fill_normal_(t, 1234, 99, 0.02)
    torch.cuda.synchronize()
    ref = oracle.fill_normal_bf16(t.numel(), 1234, 99, 0.02)
    assert np.array_equal(bits(t), ref)
    f = oracle.bf16_bits_to_f32(ref)
    assert abs(f.std() - 0.02) < 1e-3 and abs(f.mean()) < 1e-4


def test_empty_inputs_are_noops():
    """T = 0 (no routed tokens) and empty masks: every entry point returns 0
    without launching or touching outputs."""
    import ctypes as C

    from paper_2510_10302_b200 import _native

    lib = _native.load()
    s = torch.cuda.current_stream().cuda_stream
    assert lib.spmoe_router_topk(None, None, 0, 256, 8, 2, 1, None, None, None, None, None, None, s) == 0
    off = torch.zeros(9, dtype=torch.int32, device="cuda")
    assert lib.spmoe_moe_permute(None, 0, 2, 8, off.data_ptr(), None, None, s) == 0
    torch.cuda.synchronize()
    assert int(off.sum()) == 0
    slots = (C.c_int32 * 8)()
    pool = torch.zeros((1, 3 * 512 * 256), dtype=torch.bfloat16, device="cuda")
    assert lib.spmoe_expert_ffn(pool.data_ptr(), pool.shape[1], slots, 0, None, 5, 256, 512, 8, 2,
                                off.data_ptr(), None, None, None, 0, s) == 0  # empty mask
    assert lib.spmoe_moe_combine(None, None, None, 0, 256, 2, None, None, None, None, s) == 0
    assert lib.spmoe_greedy_accept(None, 512, None, 0, 4, 512, None, None, s) == 0


def test_permute_all_tokens_one_expert(oracle):
    """Degenerate routing: every token to the same experts (max tokens per
    expert) still groups stably."""
    from paper_2510_10302_b200 import kernels as K

    idx = np.tile(np.array([[5, 2]], np.int32), (72, 1))
    off, perm, inv = K.moe_permute(torch.from_numpy(idx).cuda(), 8)
    torch.cuda.synchronize()
    o2, p2, i2 = oracle.moe_permute(idx, 8)
    assert np.array_equal(bits(off), o2) and np.array_equal(bits(perm), p2) and np.array_equal(bits(inv), i2)
    o = bits(off)
    assert o[2] == 0 and o[3] - o[2] == 72 and o[6] - o[5] == 72 and o[8] == 144
