"""Layer block around the MoE (csrc/spmoe_attn.cu, K9 linear) against

* the CPU oracle (oracle/forward_oracle.c) on identical inputs: bit-exact
  (the determinism contract of include/spmoe.h), and
* plain PyTorch fp32 references of the same ops, as a sanity check of the
  contract itself: RMSNorm within one bf16 ulp; RoPE + KV append exactly
  placed (positions per sequence, other cache rows untouched) and within one
  bf16 ulp; causal GQA attention over the cache within 1e-2 of max |out|.
"""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ulps(a: torch.Tensor, b: torch.Tensor) -> int:
    ai = a.contiguous().view(torch.int16).int()
    bi = b.contiguous().view(torch.int16).int()
    return int((ai - bi).abs().max())


@pytest.mark.parametrize("rows,H", [(1, 256), (5, 4096), (63, 2048), (9, 4096)])
def test_rms_norm_matches_torch(native, rows, H):
    from paper_2510_10302_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn((rows, H), generator=g, device="cuda").to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn((H,), generator=g, device="cuda")).to(torch.bfloat16)
    got = K.rms_norm(x, w, 1e-5)
    xf = x.float()
    ref = (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()).to(torch.bfloat16)
    assert _ulps(got, ref) <= 1


def _bits(t):
    import numpy as np

    if t.dtype == torch.bfloat16:
        return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return t.contiguous().cpu().numpy()


@pytest.mark.parametrize("rows,H", [(1, 256), (5, 4096), (63, 2048)])
def test_rms_norm_bit_exact_vs_oracle(native, oracle, rows, H):
    import numpy as np

    from paper_2510_10302_b200 import kernels as K

    g = torch.Generator(device="cuda").manual_seed(rows + 7)
    x = (3 * torch.randn((rows, H), generator=g, device="cuda")).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn((H,), generator=g, device="cuda")).to(torch.bfloat16)
    assert np.array_equal(_bits(K.rms_norm(x, w, 1e-6)), oracle.rms_norm(_bits(x), _bits(w), 1e-6))


@pytest.mark.parametrize("T,K,N", [(1, 4096, 6144), (5, 4096, 4096), (9, 2048, 3072), (63, 256, 512),
                                   (5, 4096, 32000), (17, 1408, 200)])
def test_linear_bit_exact_vs_oracle(native, oracle, T, K, N):
    """K9 in all three output modes (fp32; bf16 with residual in place;
    fused RMSNorm) == the scalar oracle bit for bit; fp32 mode within fp32
    rounding of a float64 matmul."""
    import numpy as np

    from paper_2510_10302_b200 import kernels as K_

    g = torch.Generator(device="cuda").manual_seed(T * 7 + N)
    w = (0.02 * torch.randn((N, K), generator=g, device="cuda")).to(torch.bfloat16)
    x = torch.randn((T, K), generator=g, device="cuda").to(torch.bfloat16)
    y = K_.linear(x, w, f32=True)
    assert np.array_equal(_bits(y).view(np.uint32), oracle.linear(_bits(w), _bits(x), f32=True).view(np.uint32))
    ref = x.double() @ w.double().t()
    assert (y.double() - ref).abs().max().item() <= 1e-5 * ref.abs().max().item()
    r = torch.randn((T, N), generator=g, device="cuda").to(torch.bfloat16)
    want = oracle.linear(_bits(w), _bits(x), residual=_bits(r))
    K_.linear(x, w, residual=r, out=r)  # in place
    assert np.array_equal(_bits(r), want)
    nw = (1 + 0.1 * torch.randn((K,), generator=g, device="cuda")).to(torch.bfloat16)
    got = K_.linear(x, w, norm_w=nw, eps=1e-5)
    assert np.array_equal(_bits(got), oracle.linear(_bits(w), _bits(x), norm_w=_bits(nw), eps=1e-5))
    # fused norm == standalone norm followed by the projection
    assert torch.equal(got, K_.linear(K_.rms_norm(x, nw, 1e-5), w))


@pytest.mark.parametrize("B,T,nh,nkv,hd", [(1, 5, 32, 8, 128), (3, 5, 4, 2, 64), (2, 9, 16, 16, 128),
                                           (1, 63, 32, 8, 128)])
def test_rope_kv_and_attention_bit_exact_vs_oracle(native, oracle, B, T, nh, nkv, hd):
    import numpy as np

    from paper_2510_10302_b200 import kernels as K
    from paper_2510_10302_b200.model import ArchSpec, rope_tables

    g = torch.Generator(device="cuda").manual_seed(B * 10 + T)
    S = 300
    a = ArchSpec(name="t", vocab=8, hidden=nh * hd, num_layers=1, num_heads=nh, num_kv_heads=nkv, head_dim=hd,
                 ffn=8, num_experts=1, top_k=1, max_seq=S)
    cos, sin = rope_tables(a, "cuda")
    start = torch.tensor([17 + 101 * b for b in range(B)], dtype=torch.int64, device="cuda")
    kc = torch.randn((B, nkv, S, hd), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((B, nkv, S, hd), generator=g, device="cuda").to(torch.bfloat16)
    kc_o, vc_o = _bits(kc).copy(), _bits(vc).copy()
    qkv = torch.randn((B, T, (nh + 2 * nkv) * hd), generator=g, device="cuda").to(torch.bfloat16)
    q = K.rope_kv(qkv, cos, sin, start, nh, nkv, hd, kc, vc)
    q_o = oracle.rope_kv(_bits(qkv), cos.cpu().numpy(), sin.cpu().numpy(), _bits(start), nh, nkv, hd, kc_o, vc_o)
    assert np.array_equal(_bits(q), q_o)
    assert np.array_equal(_bits(kc), kc_o) and np.array_equal(_bits(vc), vc_o)
    out = K.attention_cached(q, kc, vc, start)
    assert np.array_equal(_bits(out), oracle.attention(q_o, kc_o, vc_o, _bits(start), hd ** -0.5))


def test_rope_kv_out_of_range_positions_write_nothing(native):
    """a position at or past the cache end must not write
    out of bounds; the kernel drops such rows (the engine raises first)."""
    from paper_2510_10302_b200 import kernels as K
    from paper_2510_10302_b200.model import ArchSpec, rope_tables

    a = ArchSpec(name="t", vocab=8, hidden=256, num_layers=1, num_heads=4, num_kv_heads=2, head_dim=64,
                 ffn=8, num_experts=1, top_k=1, max_seq=64)
    cos, sin = rope_tables(a, "cuda")
    big = torch.zeros((3, 2, 16, 64), dtype=torch.bfloat16, device="cuda")  # 3 "layers" back to back
    kc, vc = big[1], torch.zeros_like(big[1])
    qkv = torch.ones((1, 4, 8 * 64), dtype=torch.bfloat16, device="cuda")
    K.rope_kv(qkv, cos, sin, torch.tensor([14], dtype=torch.int64, device="cuda"), 4, 2, 64, kc, vc)
    torch.cuda.synchronize()
    assert bool((big[1, :, 14:16] != 0).any())  # positions 14, 15 written
    assert not bool(big[2].any()) and not bool(big[0].any())  # 16, 17 dropped, nothing spilled


def _ref_attention(q, kc, vc, start, T):
    """q [B, nh, T, hd]; caches [B, nkv, S, hd]; fp32 causal softmax."""
    B, nh, _, hd = q.shape
    nkv = kc.shape[1]
    out = torch.empty((B, T, nh * hd), dtype=torch.float32, device=q.device)
    for b in range(B):
        p0 = int(start[b])
        L = p0 + T
        k = kc[b, :, :L].float().repeat_interleave(nh // nkv, dim=0)  # [nh, L, hd]
        v = vc[b, :, :L].float().repeat_interleave(nh // nkv, dim=0)
        s = torch.einsum("htd,hld->htl", q[b].float(), k) / hd ** 0.5
        pos = torch.arange(T, device=q.device).view(T, 1) + p0
        s = s.masked_fill(torch.arange(L, device=q.device).view(1, L) > pos, float("-inf"))
        o = torch.einsum("htl,hld->htd", s.softmax(-1), v)  # [nh, T, hd]
        out[b] = o.permute(1, 0, 2).reshape(T, nh * hd)
    return out


@pytest.mark.parametrize("B,T,nh,nkv,hd", [(1, 5, 32, 8, 128), (3, 5, 4, 2, 64), (2, 9, 16, 16, 128),
                                           (1, 63, 32, 8, 128)])
def test_rope_kv_and_attention_match_torch(native, B, T, nh, nkv, hd):
    from paper_2510_10302_b200 import kernels as K
    from paper_2510_10302_b200.model import ArchSpec, rope_tables

    g = torch.Generator(device="cuda").manual_seed(B * 100 + T)
    S = 160
    a = ArchSpec(name="t", vocab=8, hidden=nh * hd, num_layers=1, num_heads=nh, num_kv_heads=nkv, head_dim=hd,
                 ffn=8, num_experts=1, top_k=1, max_seq=S)
    cos, sin = rope_tables(a, "cuda")
    start = torch.tensor([17 + 11 * b for b in range(B)], dtype=torch.int64, device="cuda")
    kc = torch.randn((B, nkv, S, hd), generator=g, device="cuda").to(torch.bfloat16)
    vc = torch.randn((B, nkv, S, hd), generator=g, device="cuda").to(torch.bfloat16)
    kc0, vc0 = kc.clone(), vc.clone()
    qkv = torch.randn((B, T, (nh + 2 * nkv) * hd), generator=g, device="cuda").to(torch.bfloat16)
    q = K.rope_kv(qkv, cos, sin, start, nh, nkv, hd, kc, vc)
    # reference RoPE (rotate-half, fp32, one rounding)
    qr, kr, vr = torch.split(qkv.float(), [nh * hd, nkv * hd, nkv * hd], dim=-1)
    qr, kr, vr = qr.view(B, T, nh, hd), kr.view(B, T, nkv, hd), vr.view(B, T, nkv, hd)
    pos = start.view(B, 1) + torch.arange(T, device="cuda").view(1, T)
    c, s_ = cos[pos].unsqueeze(2), sin[pos].unsqueeze(2)

    def rot(x):
        h = x.shape[-1] // 2
        return torch.cat([-x[..., h:], x[..., :h]], dim=-1)

    q_ref = (qr * c + rot(qr) * s_).to(torch.bfloat16).permute(0, 2, 1, 3)
    k_ref = (kr * c + rot(kr) * s_).to(torch.bfloat16)
    assert _ulps(q, q_ref) <= 1
    for b in range(B):
        p0 = int(start[b])
        assert _ulps(kc[b, :, p0:p0 + T], k_ref[b].permute(1, 0, 2)) <= 1
        assert torch.equal(vc[b, :, p0:p0 + T], vr[b].to(torch.bfloat16).permute(1, 0, 2))
        # rows outside the appended positions are untouched
        assert torch.equal(kc[b, :, :p0], kc0[b, :, :p0]) and torch.equal(vc[b, :, p0 + T:], vc0[b, :, p0 + T:])
    out = K.attention_cached(q, kc, vc, start)
    ref = _ref_attention(q, kc, vc, start, T)
    err = (out.float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item(), err
