"""XC: lossless exponent coding of expert blobs on the host link.

The offload tier's cost is bytes over PCIe (``IoChannel.transfer``,
``prefetch.py:45-74``; ``t_io = size / bw + overhead``, ``config.py:229-231``).
XC (format SXC5 in ``include/spmoe.h``) stores each bf16 weight as its
sign|mantissa byte plus its exponent as a 4-bit offset from the segment's
base exponent (15 = escape, exponent in a per-block exception list) in the
segment's canonical Huffman code (<= 12 bits, 32 bit-contiguous lane
substreams per 4096-value block), so a routed expert
crosses the link as ~67.5 % of its raw bytes and is expanded bit-exactly
into its HBM slot by the copy path's warp-per-block decode kernel.
Only the encoder orchestration lives here; encode / decode run on the GPU
(``csrc/spmoe_codec.cu``), there is no CPU codec in the product.
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Sequence

import numpy as np
import torch

from . import _native

XC_MAGIC = 0x35435853  # "SXC5"
XC_NSYM = 16
XC_BLOCK = 4096
XC_MAX_SEG = 4


class XcSegment(C.Structure):
    _fields_ = [
        ("n", C.c_uint64),
        ("off_lut", C.c_uint64),
        ("off_sm", C.c_uint64),
        ("off_ex", C.c_uint64),
        ("off_bofs", C.c_uint64),
        ("off_lanes", C.c_uint64),
        ("off_lbase", C.c_uint64),
        ("off_xofs", C.c_uint64),
        ("off_xrec", C.c_uint64),
        ("ex_words", C.c_uint32),
        ("n_exc", C.c_uint32),
        ("base", C.c_uint32),
        ("pad", C.c_uint32),
        ("len", C.c_uint8 * XC_NSYM),
    ]


class XcHeader(C.Structure):
    _fields_ = [
        ("magic", C.c_uint32),
        ("nseg", C.c_uint32),
        ("blob_bytes", C.c_uint64),
        ("raw_bytes", C.c_uint64),
        ("seg", XcSegment * XC_MAX_SEG),
    ]


assert C.sizeof(XcSegment) == 104 and C.sizeof(XcHeader) == 440


def expert_segments(ffn: int, hidden: int) -> list[int]:
    """An expert blob W1 | W3 | W2 codes as two segments: W1 | W3 (same
    shape and init scale: one code table, one decode launch of twice the
    blocks, so a smaller share of partial waves) and W2 (its scale differs;
    the last segment on the link, the only decode on the layer's critical
    path)."""
    return [2 * ffn * hidden, ffn * hidden]


def codec_applies(segments: Sequence[int]) -> bool:
    return 1 <= len(segments) <= XC_MAX_SEG and all(n > 0 and n % XC_BLOCK == 0 for n in segments)


def header_at(ptr: int) -> XcHeader:
    """The header of the blob at host address ``ptr`` (a copy)."""
    h = XcHeader()
    C.memmove(C.byref(h), ptr, C.sizeof(XcHeader))
    if h.magic != XC_MAGIC:
        raise ValueError("not an XC blob")
    return h


class XcEncoder:
    """GPU encoder for blobs of fixed segment sizes: ``plan(src)`` returns
    the header (blob size known), ``encode(src, hdr)`` returns the device
    blob (a view of an internal buffer, valid until the next call)."""

    def __init__(self, segments: Sequence[int], device):
        if not codec_applies(segments):
            raise ValueError(f"XC needs 1..{XC_MAX_SEG} segments of positive multiples of {XC_BLOCK} values")
        self.lib = _native.load()
        self.segments = np.asarray(segments, dtype=np.int64)
        self.device = torch.device(device)
        wb = self.lib.spmoe_xc_work_bytes(len(self.segments), self.segments.ctypes.data)
        self.work = torch.empty((max(int(wb), 4),), dtype=torch.uint8, device=self.device)
        self.blob = torch.empty((0,), dtype=torch.uint8, device=self.device)
        self.raw_elems = int(self.segments.sum())

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def plan(self, src: torch.Tensor) -> XcHeader:
        if src.dtype != torch.bfloat16 or not src.is_cuda or src.numel() != self.raw_elems:
            raise ValueError("src must be a CUDA bf16 tensor of the planned size")
        src = src.contiguous()
        hdr = XcHeader()
        _native.check("spmoe_xc_plan", self.lib.spmoe_xc_plan(
            src.data_ptr(), len(self.segments), self.segments.ctypes.data, self.work.data_ptr(),
            C.addressof(hdr), self._stream()))
        return hdr

    def encode(self, src: torch.Tensor, hdr: XcHeader) -> torch.Tensor:
        n = int(hdr.blob_bytes)
        if self.blob.numel() < n:
            self.blob = torch.empty((n,), dtype=torch.uint8, device=self.device)
        _native.check("spmoe_xc_encode", self.lib.spmoe_xc_encode(
            src.contiguous().data_ptr(), C.addressof(hdr), self.work.data_ptr(), self.blob.data_ptr(),
            self._stream()))
        return self.blob[:n]


def decode(blob: torch.Tensor, hdr: XcHeader, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Device blob -> raw bf16 (stream-ordered)."""
    if not blob.is_cuda:
        raise ValueError("blob must be on the device (there is no CPU decoder)")
    n = int(hdr.raw_bytes) // 2
    if out is None:
        out = torch.empty((n,), dtype=torch.bfloat16, device=blob.device)
    if out.numel() != n or out.dtype != torch.bfloat16:
        raise ValueError("out must be bf16 with raw_bytes / 2 elements")
    s = (stream or torch.cuda.current_stream(blob.device)).cuda_stream
    _native.call("spmoe_xc_decode", blob.data_ptr(), C.addressof(hdr), out.data_ptr(), s)
    return out
