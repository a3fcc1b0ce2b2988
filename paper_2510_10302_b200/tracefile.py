"""trace-v1 export of REAL gating scores (SURVEY.md §8 f row 4).

The reference's workload format (``trace.py:258-347``): a header
``# trace-v1 model=<name> layers=<L> experts=<E> topk=<k> shared=<S>
seed=<seed|none>`` followed by one line per (token, layer), token-major,
holding the comma-separated gating scores (a probability vector).  The B200
engine records the router's softmax over all experts for every committed
token at every layer (:meth:`SpecMoEEngine.export_trace`), so moesim's
``load_trace`` / ``simulate`` / ``sweep`` can replay real B200 routing with
calibrated timings without a GPU.
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np

HEADER = "# trace-v1"


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    x = np.asarray(logits, dtype=np.float64)
    x = x - x.max(axis=-1, keepdims=True)
    e = np.exp(x)
    return e / e.sum(axis=-1, keepdims=True)


def write_trace(path: str | Path, scores: np.ndarray, model: str, topk: int, shared: int = 0,
                seed: int | None = None) -> None:
    """``scores`` [tokens, layers, experts], each row a probability vector."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 3:
        raise ValueError("scores must be [tokens, layers, experts]")
    n, L, E = s.shape
    lines = [f"{HEADER} model={model} layers={L} experts={E} topk={topk} shared={shared} "
             f"seed={'none' if seed is None else seed}"]
    for t in range(n):
        for l in range(L):
            row = s[t, l] / math.fsum(s[t, l])
            lines.append(",".join(repr(float(v)) for v in row))
    Path(path).write_text("\n".join(lines) + "\n")


def read_trace(path: str | Path) -> tuple[dict, np.ndarray]:
    """Minimal reader (header fields, scores [tokens, layers, experts])."""
    raw = Path(path).read_text().splitlines()
    if not raw or not raw[0].startswith(HEADER):
        raise ValueError("missing trace-v1 header")
    fields = dict(p.split("=", 1) for p in raw[0][len(HEADER):].split())
    L, E = int(fields["layers"]), int(fields["experts"])
    body = [list(map(float, r.split(","))) for r in raw[1:] if r.strip()]
    if len(body) % L:
        raise ValueError("line count not a multiple of layers")
    return fields, np.asarray(body).reshape(-1, L, E)
