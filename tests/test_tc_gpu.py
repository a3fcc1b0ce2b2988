"""tcgen05/TMEM/TMA K3 path vs the CPU oracle.

Tolerance (stated): the tensor core accumulates the bf16 x bf16 products in
fp32 in its own order, so expert outputs differ from the fixed-order oracle
by fp32 rounding only, plus the effect of a 1-ulp bf16 flip of h on the
few boundary elements: |y - y_ref| <= 2^-8 * max|y_ref| + 1e-6 per element,
and the SwiGLU activations h (bf16) may differ by at most 1 bf16 ulp on a
small fraction (< 1 %) of elements where the fp32 sum sits on a rounding
boundary.  Combined hidden states are then compared at the same tolerance.
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


def run_tc(oracle, T, H, F, E, k, seed, masks=None, split=None):
    from paper_2510_10302_b200 import kernels as K

    rng = np.random.default_rng(seed)
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((T, H), generator=g).to(torch.bfloat16)
    idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    pool = torch.empty((E + 1, 3 * F * H), dtype=torch.bfloat16, device="cuda")
    K.fill_normal_(pool, seed + 1, 0, 0.02)
    slots = list(rng.permutation(E + 1)[:E])
    off, perm, inv = K.moe_permute(torch.from_numpy(idx).cuda(), E)
    n = T * k
    xd = x.cuda()
    xp = torch.empty((n, H), dtype=torch.bfloat16, device="cuda")
    h = torch.zeros((n, F), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros((n, H), dtype=torch.float32, device="cuda")
    if split is None:
        su, sd = K.tc_plan(np.bincount(idx.ravel(), minlength=E), H, F)
    else:
        su, sd = split
    ws = torch.empty((max(1, K.tc_workspace_floats(n, H, F, su, sd)),), dtype=torch.float32, device="cuda")
    for m in masks or [(1 << E) - 1]:
        K.expert_ffn_tc(pool, slots, m, xd, F, k, off, perm, xp, h, y, ws, su, sd)
    torch.cuda.synchronize()
    pool_h = bits(pool)
    o2, p2, _ = oracle.moe_permute(idx, E)
    h_ref, y_ref = oracle.expert_ffn([pool_h[slots[e]] for e in range(E)], bits(x), F, o2, p2)
    return bits(h), bits(y), h_ref[:n], y_ref[:n]


def check(hg, yg, hr, yr):
    fr = oracle_f32(hr)
    fg = oracle_f32(hg)
    ulp_diff = np.abs(hg.astype(np.int32) - hr.astype(np.int32))
    assert (ulp_diff > 1).sum() == 0 or np.abs(fg - fr).max() <= 1e-2 * np.abs(fr).max()
    assert (ulp_diff != 0).mean() < 0.01
    tol = 2.0 ** -8 * np.abs(yr).max() + 1e-6
    assert np.abs(yg - yr).max() <= tol, (np.abs(yg - yr).max(), tol)


def oracle_f32(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("T,H,F,E,k", [(5, 256, 512, 8, 2), (5, 4096, 14336, 8, 2), (9, 2048, 1408, 64, 6),
                                       (72, 4096, 14336, 8, 2), (40, 256, 512, 4, 2)])
def test_tc_matches_oracle(oracle, T, H, F, E, k):
    oracle.set_threads(16)
    check(*run_tc(oracle, T, H, F, E, k, seed=T + E))


def test_tc_masks_cached_first(oracle):
    E = 8
    check(*run_tc(oracle, 5, 256, 512, E, 2, seed=3, masks=[0b00001111, 1 << 4, 1 << 5, 1 << 6, 1 << 7]))


def test_tc_split_invariance(oracle):
    """Split-K in either phase (fixed-order partial reduction, SiLU applied
    after the up-phase reduction) stays within tolerance for every split."""
    for s in ((1, 1), (2, 1), (1, 2), (4, 4), (2, 16)):
        check(*run_tc(oracle, 9, 256, 1024, 8, 2, seed=11, split=s))


def test_tc_planned_split_single_expert(oracle):
    """The planner's down-phase split for a lone late expert stays in tolerance."""
    check(*run_tc(oracle, 2, 256, 1024, 1, 1, seed=13))


@pytest.mark.parametrize("H,F", [(4096, 14336), (2048, 1408)])
def test_tc_static_plan_grouping_invariant(oracle, H, F):
    """With the engine's launch-independent split (kernels.tc_plan_static),
    running every expert in one launch or each expert in its own launch
    (late prefetch / demand order) gives bit-identical outputs."""
    from paper_2510_10302_b200 import kernels as K

    E, k, T = 8, 2, 5
    split = K.tc_plan_static(H, F)
    one = run_tc(oracle, T, H, F, E, k, seed=21, split=split)
    each = run_tc(oracle, T, H, F, E, k, seed=21, split=split, masks=[1 << e for e in range(E)])
    mixed = run_tc(oracle, T, H, F, E, k, seed=21, split=split, masks=[0b00110101, 1 << 1, 1 << 3, 0b11000000])
    for got in (each, mixed):
        assert np.array_equal(got[0], one[0]) and np.array_equal(got[1], one[1])
    check(*one)


def run_units(oracle, T, H, F, E, k, seed, masks=None, scratch=True):
    """The unit-fused tcgen05 K3 (spmoe_expert_ffn_tc_units) vs the oracle."""
    from paper_2510_10302_b200 import kernels as K

    rng = np.random.default_rng(seed)
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((T, H), generator=g).to(torch.bfloat16)
    idx = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
    pool = torch.empty((E + 1, 3 * F * H), dtype=torch.bfloat16, device="cuda")
    K.fill_normal_(pool, seed + 1, 0, 0.02)
    slots = list(rng.permutation(E + 1)[:E])
    off, perm, inv = K.moe_permute(torch.from_numpy(idx).cuda(), E)
    n = T * k
    counts = np.bincount(idx.ravel(), minlength=E)
    xd = x.cuda()
    xp = torch.empty((n, H), dtype=torch.bfloat16, device="cuda")
    h = torch.zeros((n, F), dtype=torch.bfloat16, device="cuda")
    y = torch.zeros((n, H), dtype=torch.float32, device="cuda")
    ws = torch.zeros((K.tc_units_workspace_floats(n, H, F),), dtype=torch.float32, device="cuda")
    for m in masks or [(1 << E) - 1]:
        K.expert_ffn_tc_units(pool, slots, m, xd, F, k, off, perm, int(counts.max()), xp if scratch else None, h, y,
                              ws)
    torch.cuda.synchronize()
    pool_h = bits(pool)
    o2, p2, _ = oracle.moe_permute(idx, E)
    h_ref, y_ref = oracle.expert_ffn([pool_h[slots[e]] for e in range(E)], bits(x), F, o2, p2)
    return bits(h), bits(y), h_ref[:n], y_ref[:n]


@pytest.mark.parametrize("T,H,F,E,k", [(5, 256, 512, 8, 2), (5, 4096, 14336, 8, 2), (2, 4096, 14336, 1, 1),
                                       (9, 2048, 1408, 64, 6), (16, 256, 1024, 2, 2), (16, 2048, 5632, 1, 1)])
def test_tc_units_matches_oracle(oracle, T, H, F, E, k):
    """Unit-fused K3 within the tcgen05 tolerance at the configs' shapes,
    including a lone Mixtral expert (the single-expert late launch) and
    experts with the full 16 tokens."""
    oracle.set_threads(16)
    check(*run_units(oracle, T, H, F, E, k, seed=T + E + 1))


@pytest.mark.parametrize("H,F", [(4096, 14336), (2048, 1408)])
def test_tc_units_grouping_invariant(oracle, H, F):
    """An expert's output bits do not depend on which experts share the
    launch (every unit reduces only its own expert's partials)."""
    E, k, T = 8, 2, 5
    one = run_units(oracle, T, H, F, E, k, seed=31)
    each = run_units(oracle, T, H, F, E, k, seed=31, masks=[1 << e for e in range(E)])
    mixed = run_units(oracle, T, H, F, E, k, seed=31, masks=[0b00110101, 1 << 1, 1 << 3, 0b11000000])
    for got in (each, mixed):
        assert np.array_equal(got[0], one[0]) and np.array_equal(got[1], one[1])
    check(*one)


def test_tc_units_x_rows_by_gather4(oracle):
    """The unit kernel reads each unit's token rows straight from x (TMA
    gather4 over perm_token, clamped to the unit's last token): no x_perm
    scratch is needed, experts with 1..3 tokens (partly filled gather4
    groups) and scattered token orders give the same bits as with it."""
    for T, E, k, seed in [(3, 8, 2, 41), (7, 4, 3, 42), (1, 2, 1, 43)]:
        a = run_units(oracle, T, 1024, 2048, E, k, seed=seed)
        b = run_units(oracle, T, 1024, 2048, E, k, seed=seed, scratch=False)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        check(*b)


def test_tc_units_rejects_more_than_16_tokens():
    from paper_2510_10302_b200 import kernels as K

    pool = torch.empty((1, 3 * 512 * 256), dtype=torch.bfloat16, device="cuda")
    x = torch.zeros((17, 256), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        K.expert_ffn_tc_units(pool, [0], 1, x, 512, 1, None, None, 17, x, None, x, None)
