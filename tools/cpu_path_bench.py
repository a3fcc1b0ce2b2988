"""Time the host-core SD loop (oracle/cpu_model.py) at a bench config:
weight generation, prefill, and a few SD iterations; plus the LM kernels'
streaming rate on this host.

  python tools/cpu_path_bench.py [config] [iterations]
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    from oracle import cpu_model as CM
    from oracle import tensor_oracle as O
    from paper_2510_10302_b200.model import get_arch

    cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    arch = get_arch({"mixtral": "mixtral_8x7b", "deepseek": "deepseek_v2_lite", "qwen": "qwen15_moe_a27b",
                     "tiny": "tiny"}[cfg])
    threads = len(os.sched_getaffinity(0))
    O.set_threads(threads)
    out = {"config": cfg, "threads": threads}
    # streaming rate of the LM kernel on one big matrix
    rng = np.random.default_rng(0)
    N, K = 14336, 4096
    w = O.f32_to_bf16_bits((rng.standard_normal((N, K)) * 0.02).astype(np.float32))
    wl = O.pack_lm(w)
    x = O.f32_to_bf16_bits(rng.standard_normal((8, K)).astype(np.float32))
    for T in (1, 5):
        O.lm_linear(wl, K, x[:T], f32=True)
        t = time.perf_counter()
        for _ in range(5):
            O.lm_linear(wl, K, x[:T], f32=True)
        dt = (time.perf_counter() - t) / 5
        out[f"lm_linear_T{T}_gbs"] = N * K * 2 / dt / 1e9
    del w, wl
    t = time.perf_counter()
    cw = CM.CpuWeights.generate(arch, 1234)
    out["generate_s"] = time.perf_counter() - t
    N_ = 4
    sd = CM.CpuSD(cw, batch=1, N=N_, kv_max_seq=min(arch.max_seq, 64 + 64 * 5 + N_ + 8), cutoff=0,
                  prefetch_k=1 if arch.num_experts <= 16 else arch.top_k)
    import torch

    prompts = torch.randint(0, arch.vocab, (1, 64), generator=torch.Generator().manual_seed(1000)).numpy()
    t = time.perf_counter()
    sd.prefill(prompts)
    out["prefill_s"] = time.perf_counter() - t
    its = []
    for _ in range(iters):
        t = time.perf_counter()
        em = sd.step()
        its.append((time.perf_counter() - t, em[0]))
    out["iter_s"] = [round(a, 3) for a, _ in its]
    out["emitted"] = [e for _, e in its]
    out["tokens_per_s"] = sum(e for _, e in its) / sum(a for a, _ in its)
    print(json.dumps(out))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"cpu_path_{cfg}.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
