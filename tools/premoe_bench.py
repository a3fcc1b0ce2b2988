"""The verify layer's pre-MoE block at Mixtral-8x7B shapes, op by op (warm,
device clock by CUDA events over back-to-back reps, weights rotated over 4
layer copies so nothing is L2-resident): K9 linear qkv with the fused
RMSNorm, RoPE + KV append, cached causal GQA attention, K9 linear W_o with
the residual, the FFN RMSNorm and the K1 router -- the ≈ 0.12 ms that sits
on the critical path of every layer (profiles/r2/timeline_xc.jsonl).

python tools/premoe_bench.py [T] [kv_len]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2510_10302_b200 import kernels as K
from paper_2510_10302_b200.model import get_arch, rope_tables


def main(T=5, kv_len=200, reps=50):
    a = get_arch("mixtral_8x7b")
    dev = torch.device("cuda", 0)
    H, S = a.hidden, 512
    R = 4
    bf = torch.bfloat16
    wqkv = [torch.empty((a.qkv_dim, H), dtype=bf, device=dev) for _ in range(R)]
    wo = [torch.empty((H, a.num_heads * a.head_dim), dtype=bf, device=dev) for _ in range(R)]
    router = [torch.empty((a.num_experts, H), dtype=bf, device=dev) for _ in range(R)]
    for i in range(R):
        K.fill_normal_(wqkv[i], 10 + i, 0, 0.02)
        K.fill_normal_(wo[i], 20 + i, 0, 0.02)
        K.fill_normal_(router[i], 30 + i, 0, H ** -0.5)
    norm = torch.ones((H,), dtype=bf, device=dev)
    cos, sin = rope_tables(a, dev)
    kc = [torch.randn((1, a.num_kv_heads, S, a.head_dim), device=dev).to(bf) for _ in range(R)]
    vc = [torch.randn((1, a.num_kv_heads, S, a.head_dim), device=dev).to(bf) for _ in range(R)]
    start = torch.tensor([kv_len], dtype=torch.int64, device=dev)
    x = torch.randn((1, T, H), device=dev).to(bf)
    st = torch.cuda.current_stream()
    state = {}

    def op_qkv(i):
        state["qkv"] = K.linear(x, wqkv[i], norm_w=norm, eps=a.rms_eps)

    def op_rope(i):
        state["q"] = K.rope_kv(state["qkv"], cos, sin, start, a.num_heads, a.num_kv_heads, a.head_dim, kc[i], vc[i])

    def op_attn(i):
        state["o"] = K.attention_cached(state["q"], kc[i], vc[i], start)

    def op_wo(i):
        state["x2"] = K.linear(state["o"], wo[i], residual=x)

    def op_norm(i):
        state["xn"] = K.rms_norm(state["x2"], norm, a.rms_eps)

    def op_router(i):
        K.router_topk(state["xn"].view(T, H), router[i], a.top_k, True)

    ops = [("linear_qkv_rmsnorm", op_qkv), ("rope_kv", op_rope), ("attention", op_attn), ("linear_wo_residual", op_wo),
           ("rms_norm", op_norm), ("router_topk", op_router)]
    for i in range(R):
        for _, f in ops:
            f(i)
    torch.cuda.synchronize()
    res = {"T": T, "kv_len": kv_len}
    for name, f in ops:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for r in range(reps):
            f(r % R)
        e1.record(st)
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / reps * 1e3, 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for r in range(reps):
        for _, f in ops:
            f(r % R)
    e1.record(st)
    torch.cuda.synchronize()
    res["block_us"] = round(e0.elapsed_time(e1) / reps * 1e3, 2)
    # the same inside CUDA graphs (no host launch overhead; the engine
    # replays one graph per verify layer): per op, and the whole block
    graphs = {}
    side = torch.cuda.Stream()
    side.wait_stream(st)
    for name, f in ops + [("block", None)]:
        gs = []
        for i in range(R):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                if f is None:
                    for _, h in ops:
                        h(i)
                else:
                    f(i)
            with torch.cuda.graph(g, stream=side):
                if f is None:
                    for _, h in ops:
                        h(i)
                else:
                    f(i)
            gs.append(g)
        graphs[name] = gs
    st.wait_stream(side)
    torch.cuda.synchronize()
    for name, gs in graphs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for r in range(reps):
            gs[r % R].replay()
        e1.record(st)
        torch.cuda.synchronize()
        res["graph_" + name] = round(e0.elapsed_time(e1) / reps * 1e3, 2)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 5, int(a[1]) if len(a) > 1 else 200)
