"""XC expert-blob codec (include/spmoe.h "XC", csrc/spmoe_codec.cu).

CPU part (oracle only): the format restatement is lossless on every bf16
pattern class (Gaussian weights, zeros, denormals, inf/NaN, all 65536 bit
patterns), its header matches the documented layout, and Gaussian weights
compress to < 72 % of their raw bytes.

GPU part (``-m gpu``): the sm_100a encoder writes the oracle's blob byte for
byte; the decoder rebuilds the exact bits from oracle and GPU blobs alike,
at the test sizes and for a full Mixtral-8x7B expert (352 MB, round trip);
the native runtime's XC tier lands exact experts in their slots; and the
engine on the XC tier emits the same tokens and the same verify-MoE bits as
on the raw tier.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

BLOCK = 4096


def gaussian_bits(n, std=0.02, seed=0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(n, generator=g) * std).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def edge_bits(n, seed=1):
    """Gaussian weights with every special class sprinkled in."""
    x = gaussian_bits(n, seed=seed)
    rng = np.random.default_rng(seed)
    specials = np.array([0x0000, 0x8000, 0x0001, 0x807F, 0x7F80, 0xFF80, 0x7FC0, 0x7F7F, 0x3F80, 0x0080],
                        dtype=np.uint16)
    pos = rng.choice(n, size=min(n // 7, 5000), replace=False)
    x[pos] = specials[rng.integers(0, len(specials), size=pos.size)]
    return x


def header_fields(blob):
    h = np.frombuffer(blob[:24].tobytes(), dtype=np.uint32)
    return int(h[0]), int(h[1]), int(np.frombuffer(blob[8:16].tobytes(), np.uint64)[0]), \
        int(np.frombuffer(blob[16:24].tobytes(), np.uint64)[0])


# ----------------------------------------------------------------- CPU (oracle)
@pytest.mark.parametrize("kind", ["gauss", "edge", "all_patterns", "constant", "w2_scale"])
def test_oracle_round_trip(oracle, kind):
    if kind == "gauss":
        x, segs = gaussian_bits(3 * 8 * BLOCK), [8 * BLOCK] * 3
    elif kind == "edge":
        x, segs = edge_bits(5 * BLOCK), [2 * BLOCK, 3 * BLOCK]
    elif kind == "all_patterns":
        x, segs = np.arange(65536, dtype=np.uint16), [65536]  # 256 exponents: exceptions everywhere
    elif kind == "constant":
        x, segs = np.full(BLOCK, 0x3C00, np.uint16), [BLOCK]
    else:
        x = np.concatenate([gaussian_bits(2 * BLOCK), gaussian_bits(BLOCK, std=0.0025, seed=3)])
        segs = [BLOCK, BLOCK, BLOCK]
    blob = oracle.xc_encode(x, segs)
    magic, nseg, blob_bytes, raw_bytes = header_fields(blob)
    assert magic == 0x35435853 and nseg == len(segs)  # "SXC5"
    assert blob_bytes == blob.size and raw_bytes == 2 * x.size
    assert np.array_equal(oracle.xc_decode(blob), x)


def test_oracle_gaussian_ratio(oracle):
    x = gaussian_bits(3 * 64 * BLOCK)
    blob = oracle.xc_encode(x, [64 * BLOCK] * 3)
    # the 4096-entry decode table (16 KB per segment) is a fixed cost
    # (0.01 % of a Mixtral expert matrix, 3 % of these small segments)
    ratio = (blob.size - 3 * 16384) / (2 * x.size)
    # 8 + ~2.59 (Huffman exponent symbol) + lane lengths + exceptions
    # (~1.6e-4 of the values escape the 15-exponent window); no per-lane
    # padding (bit-contiguous substreams)
    assert ratio < 0.67, ratio


def test_oracle_rejects_partial_blocks(oracle):
    with pytest.raises(ValueError):
        oracle.xc_encode(gaussian_bits(BLOCK + 8), [BLOCK + 8])


def test_codec_header_struct_layout():
    import ctypes as C

    from paper_2510_10302_b200.codec import XcHeader, XcSegment, codec_applies, expert_segments

    assert C.sizeof(XcSegment) == 104 and C.sizeof(XcHeader) == 440
    assert codec_applies(expert_segments(14336, 4096)) and codec_applies(expert_segments(512, 256))
    assert not codec_applies([BLOCK + 1]) and not codec_applies([BLOCK] * 5)


# ----------------------------------------------------------------------- GPU
def _gpu_encode(x, segs):
    from paper_2510_10302_b200.codec import XcEncoder

    src = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    enc = XcEncoder(segs, "cuda")
    hdr = enc.plan(src)
    blob = enc.encode(src, hdr).cpu().numpy()
    return blob, hdr


def _gpu_decode(blob):
    from paper_2510_10302_b200 import codec as X

    b = np.ascontiguousarray(blob)
    hdr = X.header_at(b.ctypes.data)
    out = X.decode(torch.from_numpy(b).cuda(), hdr)
    torch.cuda.synchronize()
    return out.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["gauss", "edge", "all_patterns", "constant", "w2_scale", "tiny_expert"])
def test_gpu_encoder_matches_oracle_bytes(oracle, native, kind):
    if kind == "gauss":
        x, segs = gaussian_bits(3 * 8 * BLOCK), [8 * BLOCK] * 3
    elif kind == "edge":
        x, segs = edge_bits(5 * BLOCK), [2 * BLOCK, 3 * BLOCK]
    elif kind == "all_patterns":
        x, segs = np.arange(65536, dtype=np.uint16), [65536]
    elif kind == "constant":
        x, segs = np.full(BLOCK, 0x3C00, np.uint16), [BLOCK]
    elif kind == "w2_scale":
        x = np.concatenate([gaussian_bits(2 * BLOCK), gaussian_bits(BLOCK, std=0.0025, seed=3)])
        segs = [BLOCK, BLOCK, BLOCK]
    else:  # the tiny config's expert blob shape: 3 x 512 x 256
        x, segs = gaussian_bits(3 * 512 * 256, seed=9), [512 * 256] * 3
    ref = oracle.xc_encode(x, segs)
    got, hdr = _gpu_encode(x, segs)
    assert int(hdr.blob_bytes) == ref.size
    assert np.array_equal(got, ref), "GPU blob differs from the oracle's"
    assert np.array_equal(_gpu_decode(ref), x)
    assert np.array_equal(_gpu_decode(got), x)


@pytest.mark.gpu
def test_gpu_full_mixtral_expert_round_trip(native):
    """A whole Mixtral-8x7B expert (W1|W3|W2, 352 MB) generated by the
    model's own init: decode(encode(x)) == x bit for bit, and the blob is
    < 72 % of the raw bytes.  Also times the decoder (HBM-bound)."""
    from paper_2510_10302_b200 import codec as X
    from paper_2510_10302_b200.model import fill_expert_blob, get_arch

    a = get_arch("mixtral_8x7b")
    src = torch.empty((a.expert_elems,), dtype=torch.bfloat16, device="cuda")
    fill_expert_blob(src, a, 1234, 77)
    enc = X.XcEncoder(X.expert_segments(a.ffn, a.hidden), "cuda")
    hdr = enc.plan(src)
    blob = enc.encode(src, hdr)
    assert int(hdr.blob_bytes) < 0.69 * a.expert_bytes
    out = torch.empty_like(src)
    X.decode(blob, hdr, out)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), src.view(torch.int16))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        X.decode(blob, hdr, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    gbs = (int(hdr.blob_bytes) + a.expert_bytes) / (ms / 1e3) / 1e9
    print(f"xc decode: {ms:.3f} ms per expert, {gbs:.0f} GB/s (read blob + write raw)")
    assert gbs > 1000


@pytest.mark.gpu
def test_runtime_xc_tier_lands_exact_experts(oracle, native):
    """Demand loads through the native runtime's XC tier (staging ring of 2,
    more experts than buffers) put the exact raw expert bits in each slot."""
    from paper_2510_10302_b200.cache import ExpertId, NativeExpertCache

    L, E, segs = 2, 4, [BLOCK * 16] * 3  # large enough that the 16 KB table per segment amortises
    raw = [gaussian_bits(sum(segs), seed=s) for s in range(L * E)]
    blobs = [oracle.xc_encode(r, segs) for r in raw]
    stride = (max(b.size for b in blobs) + 4095) // 4096 * 4096
    host = torch.zeros((L * E, stride), dtype=torch.uint8).pin_memory()
    for i, b in enumerate(blobs):
        host[i, : b.size] = torch.from_numpy(b)
    slot_bytes = 2 * sum(segs)
    pool = torch.zeros((3, slot_bytes // 2), dtype=torch.bfloat16, device="cuda")
    copy, dec = torch.cuda.Stream(), torch.cuda.Stream()
    staging = torch.empty((2 * stride,), dtype=torch.uint8, device="cuda")
    c = NativeExpertCache(3, L, E, dev_pool_ptr=pool.data_ptr(), host_pool_ptr=host.data_ptr(),
                          slot_bytes=slot_bytes, copy_stream_ptr=copy.cuda_stream)
    try:
        c.set_codec(stride, staging.data_ptr(), stride, 2, dec.cuda_stream)
        c.decode_timing(True)
        cur = torch.cuda.current_stream().cuda_stream
        for l, e in [(0, 1), (1, 3), (0, 2), (1, 0), (0, 1), (1, 2)]:
            s = c.demand_load([ExpertId(l, e)])[0]
            c.wait_slot(s, cur)
            got = pool[s].view(torch.int16).cpu().numpy().view(np.uint16)
            assert np.array_equal(got, raw[l * E + e]), (l, e)
            c.mark_read(s, cur)
        # capacity 3: every one of the six loads misses (LRU evicts the
        # oldest), so the link carried exactly the six blobs
        wire = c.wire_bytes()
        seq = [(0, 1), (1, 3), (0, 2), (1, 0), (0, 1), (1, 2)]
        assert wire["demand"] == sum(blobs[l * E + e].size for l, e in seq)
        log = c.transfer_log()
        assert all(r["wire_bytes"] < slot_bytes for r in log)
        # one timed decode per segment of every load; bytes = blob + raw
        st = c.decode_stats()
        assert st["launches"] == 3 * len(seq) and st["ms"] > 0
        assert st["bytes"] == wire["demand"] + len(seq) * slot_bytes
        assert c.decode_stats()["launches"] == 0
    finally:
        torch.cuda.synchronize()
        c.close()


@pytest.mark.gpu
def test_engine_xc_tier_equals_raw_tier(oracle):
    """Same model, policy and prompts on the XC and the raw host tier:
    identical tokens, identical cache decisions, identical verify-MoE bits;
    the XC tier moves fewer bytes over the link."""
    from test_engine_gpu import check_layer_captures, make_engine, prompts

    out = {}
    for codec in ("xc", None):
        eng = make_engine(capture=(0, 3), host_codec=codec)
        try:
            assert eng.host_pool.codec == codec
            eng.prefill(prompts(1))
            em = [eng.step() for _ in range(4)]
            torch.cuda.synchronize()
            check_layer_captures(eng, oracle)
            rep = eng.report()
            caps = [(c["layer"], c["out"].view(torch.int16).cpu().numpy()) for c in eng.captures if "layer" in c]
            out[codec] = (em, [list(s) for s in eng.seqs], eng.decisions, caps, rep.extras, rep.counters)
        finally:
            eng.close()
    xc, raw = out["xc"], out[None]
    assert xc[0] == raw[0] and xc[1] == raw[1] and xc[2] == raw[2]
    assert len(xc[3]) == len(raw[3]) and all(a[0] == b[0] and np.array_equal(a[1], b[1]) for a, b in zip(xc[3], raw[3]))
    assert xc[5] == raw[5]
    assert xc[4]["h2d_bytes"] == raw[4]["h2d_bytes"]
    assert xc[4]["h2d_wire_bytes"] < 0.75 * raw[4]["h2d_wire_bytes"]
    assert raw[4]["h2d_wire_bytes"] == raw[4]["h2d_bytes"]
