"""Single-launch (cooperative, grid-barrier) tcgen05 K3 vs the CPU oracle,
same tolerance as tests/test_tc_gpu.py, and vs the two-launch tcgen05 path
(identical tile order and accumulation -> identical bits)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def bits(t):
    if t.dtype == torch.bfloat16:
        return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return t.contiguous().cpu().numpy()


def run(oracle, T, H, F, E, k, seed, split_dn=None, masks=None):
    from paper_2510_10302_b200 import kernels as K

    rng = np.random.default_rng(seed)
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((T, H), generator=g).to(torch.bfloat16).cuda()
    idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    pool = torch.empty((E + 1, 3 * F * H), dtype=torch.bfloat16, device="cuda")
    K.fill_normal_(pool, seed + 1, 0, 0.02)
    slots = list(rng.permutation(E + 1)[:E])
    off, perm, inv = K.moe_permute(torch.from_numpy(idx).cuda(), E)
    n = T * k
    sd = K.tc_plan(np.bincount(idx.ravel(), minlength=E), H, F)[1] if split_dn is None else split_dn
    xp = torch.empty((n, H), dtype=torch.bfloat16, device="cuda")
    ws = torch.empty((max(1, sd * n * H),), dtype=torch.float32, device="cuda")
    sync = torch.zeros((1,), dtype=torch.int32, device="cuda")
    hf = torch.zeros((n, F), dtype=torch.bfloat16, device="cuda")
    yf = torch.zeros((n, H), dtype=torch.float32, device="cuda")
    for m in masks or [(1 << E) - 1]:
        K.expert_ffn_tc_fused(pool, slots, m, x, F, k, off, perm, xp, hf, yf, ws, sd, sync)
    h2 = torch.zeros_like(hf)
    y2 = torch.zeros_like(yf)
    for m in masks or [(1 << E) - 1]:
        K.expert_ffn_tc(pool, slots, m, x, F, k, off, perm, xp, h2, y2, ws, 1, sd)
    torch.cuda.synchronize()
    o2, p2, _ = oracle.moe_permute(idx, E)
    pool_h = bits(pool)
    h_ref, y_ref = oracle.expert_ffn([pool_h[slots[e]] for e in range(E)], bits(x), F, o2, p2)
    return bits(hf), bits(yf), bits(h2), bits(y2), h_ref[:n], y_ref[:n]


@pytest.mark.parametrize("T,H,F,E,k", [(5, 256, 512, 8, 2), (5, 4096, 14336, 8, 2), (9, 2048, 1408, 64, 6),
                                       (72, 4096, 14336, 8, 2), (2, 4096, 14336, 1, 1)])
def test_fused_matches_oracle_and_two_launch(oracle, T, H, F, E, k):
    oracle.set_threads(16)
    hf, yf, h2, y2, hr, yr = run(oracle, T, H, F, E, k, seed=T + 3 * E)
    assert np.array_equal(hf, h2) and np.array_equal(yf.view(np.uint32), y2.view(np.uint32))
    assert np.abs(yf - yr).max() <= 2.0 ** -8 * np.abs(yr).max() + 1e-6
    assert (hf != hr).mean() < 0.01


def test_fused_masks_and_splits(oracle):
    for sd in (1, 2, 4):
        hf, yf, h2, y2, hr, yr = run(oracle, 5, 256, 1024, 8, 2, seed=7, split_dn=sd,
                                     masks=[0b00001111, 1 << 4, 1 << 5, 1 << 6, 1 << 7])
        assert np.array_equal(yf.view(np.uint32), y2.view(np.uint32))
        assert np.abs(yf - yr).max() <= 2.0 ** -8 * np.abs(yr).max() + 1e-6
