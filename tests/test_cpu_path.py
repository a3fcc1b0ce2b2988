"""The lane-major CPU path (oracle/cpu_path.c: SIMD layout of the
determinism contract, the code bench.py times as the reference arm and the
end-to-end tests run as the SD-loop oracle) against the scalar oracles
(spmoe_oracle.c / forward_oracle.c) bit for bit, on CPU."""

from __future__ import annotations

import numpy as np
import pytest


def rand_bf16(oracle, rng, shape, scale=1.0):
    return oracle.f32_to_bf16_bits((rng.standard_normal(shape) * scale).astype(np.float32))


@pytest.mark.parametrize("K,N,T", [(256, 40, 1), (512, 33, 5), (1408, 24, 3), (4096, 16, 9), (1024, 8, 17)])
def test_lm_linear_equals_scalar(oracle, K, N, T):
    rng = np.random.default_rng(K + N + T)
    w = rand_bf16(oracle, rng, (N, K), 0.05)
    x = rand_bf16(oracle, rng, (T, K))
    wl = oracle.pack_lm(w)
    assert wl.shape == (N, (K + 255) // 256 * 256)
    assert np.array_equal(oracle.lm_linear(wl, K, x, f32=True).view(np.uint32),
                          oracle.linear(w, x, f32=True).view(np.uint32))
    r = rand_bf16(oracle, rng, (T, N))
    assert np.array_equal(oracle.lm_linear(wl, K, x, residual=r), oracle.linear(w, x, residual=r))
    g = rand_bf16(oracle, rng, (K,), 0.3)
    assert np.array_equal(oracle.lm_linear(wl, K, x, norm_w=g, eps=1e-5),
                          oracle.linear(w, x, norm_w=g, eps=1e-5))
    # K9 = dot_fixed per element
    y = oracle.linear(w, x, f32=True)
    assert y[T - 1, N - 1] == np.float32(oracle.dot_fixed(w[N - 1], x[T - 1]))


@pytest.mark.parametrize("H,F,n", [(256, 512, 1), (256, 512, 6), (2048, 1408, 3)])
def test_lm_expert_ffn_equals_scalar(oracle, H, F, n):
    rng = np.random.default_rng(H + F + n)
    blob = rand_bf16(oracle, rng, (3 * F * H,), 0.02)
    x = rand_bf16(oracle, rng, (n + 2, H))
    perm = rng.permutation(n + 2)[:n].astype(np.int32)
    h_lm, y_lm = oracle.lm_expert_ffn(oracle.pack_blob(blob, H, F), H, F, x, perm)
    off = np.array([0, n], np.int32)
    h_s, y_s = oracle.expert_ffn([blob], x, F, off, perm)
    assert np.array_equal(h_lm, h_s[:n])
    assert np.array_equal(y_lm.view(np.uint32), y_s[:n].view(np.uint32))


def test_rms_norm_scale_contract(oracle):
    rng = np.random.default_rng(0)
    x = rand_bf16(oracle, rng, (3, 512))
    w = np.full((512,), 0x3F80, np.uint16)  # 1.0
    out = oracle.rms_norm(x, w, 1e-5)
    xf = oracle.bf16_bits_to_f32(x)
    ref = xf / np.sqrt((xf.astype(np.float64) ** 2).mean(-1, keepdims=True) + 1e-5)
    got = oracle.bf16_bits_to_f32(out)
    assert np.abs(got - ref).max() <= 2 ** -7 * np.abs(ref).max()


def test_attention_matches_float64_softmax(oracle):
    """Contract sanity: the fixed-order attention equals a float64 softmax
    attention within fp32/bf16 rounding (the bit-level pin is the GPU test)."""
    rng = np.random.default_rng(1)
    B, T, nh, nkv, hd, S = 1, 3, 4, 2, 64, 32
    cos = np.ones((S, hd), np.float32)
    sin = np.zeros((S, hd), np.float32)
    kc = np.zeros((B, nkv, S, hd), np.uint16)
    vc = np.zeros((B, nkv, S, hd), np.uint16)
    start = np.array([10], np.int64)
    hist = rand_bf16(oracle, rng, (B, 10, (nh + 2 * nkv) * hd))
    oracle.rope_kv(hist, cos, sin, np.array([0], np.int64), nh, nkv, hd, kc, vc)
    qkv = rand_bf16(oracle, rng, (B, T, (nh + 2 * nkv) * hd))
    q = oracle.rope_kv(qkv, cos, sin, start, nh, nkv, hd, kc, vc)
    out = oracle.bf16_bits_to_f32(oracle.attention(q, kc, vc, start, hd ** -0.5)).reshape(B, T, nh, hd)
    qf = oracle.bf16_bits_to_f32(q).astype(np.float64)
    kf = oracle.bf16_bits_to_f32(kc).astype(np.float64)
    vf = oracle.bf16_bits_to_f32(vc).astype(np.float64)
    for t in range(T):
        for h in range(nh):
            kh = h // (nh // nkv)
            s = kf[0, kh, : 11 + t] @ qf[0, h, t] * hd ** -0.5
            p = np.exp(s - s.max())
            ref = (p / p.sum()) @ vf[0, kh, : 11 + t]
            assert np.abs(out[0, t, h] - ref).max() <= 1e-2 * max(1e-3, np.abs(ref).max())


def test_cpu_model_restates_model_helpers():
    """The CPU SD loop's restated init helpers equal the product's."""
    from oracle import cpu_model as CM
    from paper_2510_10302_b200 import model as M

    for ids in [(1234,), (1234, 4, 3), (7, 2, 31, 10_000)]:
        assert CM.tensor_seed(*ids) == M.tensor_seed(*ids)
    assert (CM.K_EMBED, CM.K_BASE, CM.K_LMHEAD) == (M.K_EMBED, M.K_BASE, M.K_LMHEAD)
    a = M.get_arch("tiny")
    c1, s1 = CM.rope_tables(a.head_dim, a.rope_theta, a.max_seq)
    c2, s2 = M.rope_tables_host(a)
    assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
    r = np.random.default_rng(0).standard_normal((16, 64)).astype(np.float32)
    assert CM.gate_mass(r, 4, False) == M.gate_mass(r, 4, False)
    assert CM.gate_mass(r, 4, True) == 1.0


def test_cpu_sd_loop_tiny_runs(oracle):
    """The host SD loop on the CPU-generated tiny pair: tokens emitted per
    iteration in [1, N+1], reproducible."""
    from oracle import cpu_model as CM
    from paper_2510_10302_b200.model import get_arch

    a = get_arch("tiny")
    w = CM.CpuWeights.generate(a, 1234)
    outs = []
    for _ in range(2):
        sd = CM.CpuSD(w, batch=1, N=4, kv_max_seq=64, cutoff=3)
        sd.prefill(np.arange(12, dtype=np.int64).reshape(1, 12) * 37 % a.vocab)
        em = [sd.step()[0] for _ in range(4)]
        assert all(1 <= e <= 5 for e in em)
        assert len(sd.predictions) == 4 * 4 * 4  # steps x layers <= cutoff x iterations
        outs.append(list(sd.seqs[0]))
    assert outs[0] == outs[1]
