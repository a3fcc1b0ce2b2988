#!/usr/bin/env python
"""Benchmark of the SP-MoE verification-time expert path on B200.

Default workload (BASELINE.json configs[1]): Mixtral-8x7B-shaped target
(random init, bf16) with a small dense draft (shares the target's embedding,
attention and lm_head; FFN = mean of the layer's experts), expert-cache budget
25 % of the routed experts (64 of 256 slots) with the other 75 % offloaded to
pinned host memory, draft length N=4, batch 1, SP-MoE draft_prefetch policy.

A *step* is one SD iteration (draft N tokens with draft-guided prediction +
asynchronous prefetch, verify N+1 tokens through all 32 layers with
demand loads, greedy acceptance).  ``value`` = emitted tokens/s over the
timed steps (device time by CUDA events, max over ranks; weak scaling: one
independent request stream per GPU); ``e2e`` = the same through the public
``SpecMoEEngine.step`` API by wall clock, including per-step host->device
token inputs and the device->host read of the accepted tokens.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config mixtral|deepseek|qwen|tiny] [--batch B] [--draft-length N]

Multi-GPU: launched by torch.distributed.run, one rank per GPU over NCCL
(barrier + max-over-ranks timing only; there is no data-path collective).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TPOT ms and tokens/s, Mixtral-8x7B SD+offload; verify-MoE HBM GB/s; H2D GB/s"
UNIT = "tokens/s"
CPU_SAMPLE_LAYERS = 4

CONFIGS = {
    # configs[1]: the headline
    # 128-token synthetic prompts
    "mixtral": dict(arch="mixtral_8x7b", budget=0.25, N=4, batch=1, prompt=128),
    "deepseek": dict(arch="deepseek_v2_lite", budget=0.25, N=4, batch=1, prompt=128),
    "qwen": dict(arch="qwen15_moe_a27b", budget=0.25, N=4, batch=1, prompt=128),
    "tiny": dict(arch="tiny", budget=0.375, N=4, batch=1, prompt=16),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.f = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def h2d_peak_gbs(torch, nbytes=1 << 30, reps=5) -> float:
    """Pinned host -> HBM copy bandwidth on this box (best of ``reps``)."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            d.copy_(h, non_blocking=True)
            b.record(s)
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    del h, d
    return best


# ---------------------------------------------------------------------------
# CPU restatement (oracle port) of the same path: the reference arm and the
# cpu_baseline leg.  Executes oracle/ only here, as the timed CPU baseline.
# ---------------------------------------------------------------------------
def kv_max_seq(arch, cfg) -> int:
    """The engine's KV capacity for this config (SpecMoEEngine max_seq)."""
    N = cfg["N"]
    return min(arch.max_seq, cfg["prompt"] + 64 * (N + 1) + N + 8)


def bench_prompts(arch, cfg, rank):
    import torch

    g = torch.Generator().manual_seed(1000 + rank)
    return torch.randint(0, arch.vocab, (cfg["batch"], cfg["prompt"]), generator=g)


def cpu_sd(arch, cfg, threads, layers=None, log_fn=None):
    """The SD loop on the host cores (oracle/cpu_model.py: the CPU
    restatement of the engine's draft forward, predictor, verify MoE and
    greedy acceptance on the same determinism contract), on weights
    regenerated on the CPU with the engine's counter-hash streams -- the
    same model bit for bit (tests/test_e2e_gpu.py), no GPU involved.
    ``layers``: keep only the first ``layers`` decoder layers (bounded
    sample)."""
    from dataclasses import replace

    from oracle import cpu_model as CM
    from oracle import tensor_oracle as O

    O.set_threads(threads)
    a = replace(arch, num_layers=layers) if layers else arch
    t0 = time.perf_counter()
    w = CM.CpuWeights.generate(a, 1234)
    t_gen = time.perf_counter() - t0
    pk = 1 if arch.num_experts <= 16 else arch.top_k
    # the drafting-stage predictor runs at layer 0 (the cutoff the GPU arm's
    # recalibration settles on at this config); it is a few router dots
    sd = CM.CpuSD(w, batch=cfg["batch"], N=cfg["N"], kv_max_seq=kv_max_seq(arch, cfg), cutoff=0, prefetch_k=pk)
    t0 = time.perf_counter()
    sd.prefill(bench_prompts(arch, cfg, 0).numpy())
    t_pre = time.perf_counter() - t0
    if log_fn:
        log_fn(f"[cpu] {a.num_layers}-layer model generated in {t_gen:.1f}s, prefill {t_pre:.1f}s, {threads} threads")
    return sd, t_gen, t_pre


def host_threads() -> int:
    try:  # the CPU path may use every host core, not just the GPU's socket
        os.sched_setaffinity(0, range(os.cpu_count() or 1))
    except OSError:
        pass
    return len(os.sched_getaffinity(0))


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU restatement of the path (oracle port; the
    reference package is a Python simulator with no tensor path and cannot
    travel to the GPU box) on all host threads.  Every step is one FULL SD
    iteration of the configured model (all layers: N draft steps with the
    draft-guided predictor, the N+1-token verify through every MoE layer,
    lm_head, greedy acceptance); tokens come from this CPU loop itself."""
    from paper_2510_10302_b200.model import get_arch

    if rank != 0:
        return
    arch = get_arch(cfg["arch"])
    threads = host_threads()
    sd, t_gen, t_pre = cpu_sd(arch, cfg, threads, log_fn=log)
    for _ in range(args.warmup):
        sd.step()
    emitted = 0
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        emitted += sum(sd.step())
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = emitted / total
    it_ms = total / args.steps * 1e3
    B, N = cfg["batch"], cfg["N"]
    sample = (f"{args.steps} timed full SD iterations (after {args.warmup} warm-up) of {arch.name}: all "
              f"{arch.num_layers} layers, N={N} draft steps + {N + 1}-token verify + lm_head + greedy acceptance, "
              f"batch {B}, prompt {cfg['prompt']}; oracle/cpu_model.py on {threads} threads; "
              f"{emitted / args.steps / B:.2f} tokens/iteration from this CPU loop")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": it_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16 weights, fp32 accumulate", "data": "synthetic",
        "config": {"workload": f"{args.config}: {arch.name} SD verify path, N={N}, batch {B}",
                   "prompt_len": cfg["prompt"]},
        "tpot_ms": total * 1e3 / (emitted / B) if emitted else None,
        "tokens_emitted": emitted,
        "setup_s": {"generate_weights": t_gen, "prefill": t_pre},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def spawn_ranks(args) -> int:
    """``--gpus N`` without a torchrun environment: launch N ranks of this
    script through torch.distributed.run on 127.0.0.1 (one process per
    GPU), forward its exit status.  Rank 0 prints the JSON line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # rank/channel count visible in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py")] + sys.argv[1:]
    log(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=23)  # ~100 emitted tokens
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--draft-length", type=int, default=None)
    ap.add_argument("--budget", type=float, default=None, help="fraction of routed experts resident in HBM")
    ap.add_argument("--policy", default="draft_prefetch")
    ap.add_argument("--cutoff", type=int, default=None, help="explicit cutoff layer (default: solver)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-event-pass", dest="event_pass", action="store_false",
                    help="skip the 2 extra steps that time the roofline kernels with CUDA events")
    ap.add_argument("--ffn-impl", default="auto", choices=["auto", "tcgen05", "cuda_core"])
    ap.add_argument("--tc-min-tokens", type=int, default=None,
                    help="experts with fewer routed tokens take the CUDA-core K3 (default 1: tcgen05 for every expert)")
    ap.add_argument("--host-codec", default="xc", choices=["xc", "none"],
                    help="host-tier expert encoding: xc (lossless exponent coding) or raw bf16")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.draft_length:
        cfg["N"] = args.draft_length
    if args.budget:
        cfg["budget"] = args.budget
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}")
        sys.exit(2)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec
    from paper_2510_10302_b200 import kernels as K
    from paper_2510_10302_b200.calibrate import b200_timings
    from paper_2510_10302_b200.engine import SpecMoEEngine
    from paper_2510_10302_b200.model import get_arch

    # SPMOE_BENCH_SHARE_GPU=1 (test hook): every rank on cuda:0 over gloo, so
    # the replica plumbing (pool roles, placement plan, shared-pool attach,
    # max-over-ranks reduction) can be exercised on a one-GPU box
    share_gpu = os.environ.get("SPMOE_BENCH_SHARE_GPU") == "1"
    dev_index = 0 if share_gpu else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    arch = get_arch(cfg["arch"])
    E_all = arch.num_layers * arch.num_experts
    capacity = max(arch.num_experts, int(round(cfg["budget"] * E_all)))
    if world > 1:
        dist.barrier()  # every rank copies at once: the concurrent host-link peak
    peak_h2d = h2d_peak_gbs(torch)
    hw = HardwareSpec(gpu_memory=183_359 * 2**20, peak_non_expert_memory=24 * 10**9, pcie_bandwidth=peak_h2d * 1e9,
                      name="b200")
    timings = b200_timings(arch, hw)
    policy = PolicySpec(policy=Policy(args.policy), prefetch_k=1 if arch.num_experts <= 16 else arch.top_k,
                        draft_length=cfg["N"], acceptance_rate=1.0, seed=1234, cutoff_layer=args.cutoff,
                        cache_capacity_experts=capacity)
    t_setup = time.perf_counter()
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    # replicas on one box share one pinned host expert pool per NUMA node
    # through /dev/shm; each process runs on its GPU's socket
    from paper_2510_10302_b200.replicas import (bind_to_node, gpu_numa_node, mem_available_bytes, numa_pool_roles,
                                                plan_host_pools, shm_free_bytes)

    node = gpu_numa_node(dev_index)
    bind_to_node(node)
    share, leader, distinct = None, True, None
    if local_world > 1:
        nodes = [node] * world
        if world > 1:
            allnodes = [None] * world
            dist.all_gather_object(allnodes, (local, node))
            nodes = [n for _, n in sorted(allnodes)][:local_world]
        node, leader = numa_pool_roles(nodes, local)
        # rank 0 decides for the box (before any pool exists): shared shm
        # pools if they fit, else private pinned pools bounded by free RAM
        wire = 0.72 if args.host_codec != "none" else 1.0  # XC blob ~0.673 of raw
        decision = [plan_host_pools(len(set(nodes)), int(wire * E_all * arch.expert_bytes), local_world, E_all,
                                    shm_free_bytes(), mem_available_bytes())]
        if world > 1:
            dist.broadcast_object_list(decision, src=0)
        use_shared, distinct = decision[0]
        if use_shared:
            share = f"{arch.name}_s1234_{os.environ.get('MASTER_PORT', '0')}_n{node}"
        else:
            leader = True
            log(f"[bench] /dev/shm too small for shared pools: private pinned pools, distinct rows={distinct}")
    eng = SpecMoEEngine(arch, hw, timings, policy, batch=cfg["batch"], max_tokens=cfg["prompt"] + 96 * (cfg["N"] + 1),
                        window_tokens=cfg["N"], host_share=share, host_leader=leader, host_distinct=distinct,
                        ffn_impl=args.ffn_impl, host_codec=None if args.host_codec == "none" else "xc",
                        tc_min_tokens=args.tc_min_tokens)
    prompts = bench_prompts(arch, cfg, rank)
    eng.prefill(prompts)
    log(f"[bench] setup {time.perf_counter() - t_setup:.1f}s capacity={capacity} cutoff={eng.cutoff} "
        f"h2d_peak={peak_h2d:.1f}GB/s timings={timings}")
    for _ in range(args.warmup):
        eng.step()
    torch.cuda.synchronize()
    # cutoff model recalibrated from this GPU's measured draft/verify layer
    # times and host-link copy time
    cutoff_analytic = eng.cutoff
    measured = eng.recalibrate()
    eng.step()
    torch.cuda.synchronize()
    log(f"[bench] measured timings {measured} -> cutoff {cutoff_analytic} -> {eng.cutoff}")
    eng._reset_run_state()
    eng.cache.reset_stats()
    eng.cache.clear_log()
    # per-launch kernel durations for the rooflines: device-clock spans
    # (globaltimer, first CTA start -> last CTA end) -- CUDA events around
    # launches are skewed by ~30 us per pair while the host link is saturated
    # (profiles/r2_event_skew_probe.txt); an event-timed pass follows below
    eng.time_k3 = True
    if eng.host_pool.codec:
        eng.cache.decode_stats()  # drop warm-up records
        eng.cache.decode_timing("device")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
    clocks.start()
    launches0 = K.LAUNCHES["count"]
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    prof_range = os.environ.get("SPMOE_PROFILE_RANGE") == "1"
    if prof_range:
        torch.cuda.profiler.start()
    e0.record(st)
    emitted = 0
    for _ in range(args.steps):
        emitted += sum(eng.step())
    e1.record(st)
    if prof_range:
        torch.cuda.profiler.stop()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = K.LAUNCHES["count"] - launches0
    dev_ms = e0.elapsed_time(e1)
    rep = eng.report(wall_s=wall)
    roof = eng.k3_roofline()
    dec = eng.cache.decode_stats() if eng.host_pool.codec else None
    # the same kernels timed with CUDA events on their streams (2 untimed
    # extra steps, outside the timed region): the event-based figures
    ev_k3, ev_dec = None, None
    if args.event_pass:
        eng._reset_run_state()
        eng.time_k3 = "events"
        if eng.host_pool.codec:
            eng.cache.decode_timing("events")
        for _ in range(2):
            eng.step()
        torch.cuda.synchronize()
        r2 = eng.k3_roofline()
        ev_k3 = r2.get("events_ms_per_launch")
        if ev_k3:
            ev_k3 = {"ms_per_launch": ev_k3, "achieved": r2["bytes_per_launch"] / (ev_k3 / 1e3) / 1e9}
        if eng.host_pool.codec:
            d2 = eng.cache.decode_stats()
            eng.cache.decode_timing(False)
            if d2["launches"]:
                ev_dec = {"ms_per_launch": d2["ms"] / d2["launches"], "achieved": d2["gbs"]}
        eng.time_k3 = False
    per_rank = None
    stats = torch.tensor([dev_ms, wall, float(emitted)], dtype=torch.float64, device="cpu" if share_gpu else "cuda")
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"h2d_peak_gbs": peak_h2d, "h2d_gbs": rep.extras.get("h2d_wire_gbs"),
                                          "link_busy_frac": rep.extras.get("link_busy_frac"),
                                          "tokens": emitted, "device_ms": dev_ms})
        dev_ms, wall, emitted_all = float(mx[0]), float(mx[1]), float(sm[2])
    else:
        emitted_all = float(emitted)
    value = emitted_all / (dev_ms / 1e3)
    e2e = emitted_all / wall
    peaks = measured_peaks()
    B, N = cfg["batch"], cfg["N"]
    # per-step host<->device bytes of the public step() API: int64 token /
    # position inputs (first[B,2], start[B], last[B,1], vstart[B]) and the
    # int32 result [B,2] + drafts [B,N]
    h2d_step = 8 * B * (2 + 1 + 1 + 1)
    d2h_step = 4 * B * (2 + N)
    ex = rep.extras
    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights, seeded random prompts)",
        "config": {
            "workload": f"{args.config}: {arch.name} target + dense draft, SD N={N}, batch {B}/GPU, "
                        f"expert budget {cfg['budget']:.0%} ({capacity}/{E_all} slots), policy {args.policy}",
            "global_batch": B * world,
            "prompt_len": cfg["prompt"],
            "l2": "inputs larger than L2: each step streams >=20 GB of expert weights (126 MB L2)",
            "parallelism": f"replicas x{world} (independent SD streams, per-GPU caches, host pool per NUMA node)",
            "numa_node": node,
        },
        "tpot_ms": dev_ms / args.steps / (emitted / args.steps / B) if emitted else None,
        "tokens_emitted": emitted_all,
        "acceptance_rate": ex.get("acceptance_rate"),
        "hit_rate": rep.hit_rate,
        "cutoff_layer": eng.cutoff,
        "cutoff_calibration": {
            "analytic_cutoff": cutoff_analytic,
            "measured_timings_ms": {"t_comp_draft": measured.t_comp_draft * 1e3,
                                    "t_comp_target": measured.t_comp_target * 1e3,
                                    "t_io_expert": measured.t_io_expert * 1e3,
                                    "t_predict": measured.t_predict * 1e3},
            "window_tokens": cfg["N"],
            "cutoff_source": getattr(eng, "cutoff_source", None),
            "k_eff_measured": getattr(eng, "k_eff", None),
        },
        "latency_breakdown": rep.latency_breakdown,
        "verify_moe_hbm_gbs": roof.get("achieved_gbs"),
        # host link: bytes that crossed it per second of copy time, against
        # the pinned H2D peak measured on this box; with the XC tier the
        # decoded expert bytes per copy second are higher by 1 / wire_ratio
        "h2d_gbs": ex.get("h2d_wire_gbs"),
        "h2d_peak_gbs": peak_h2d,
        # world > 1: each rank's pinned peak measured concurrently with all
        # others (shared host DRAM / PCIe switches) and its timed-region link use
        "per_rank": per_rank if world > 1 else None,
        "h2d_frac": (ex.get("h2d_wire_gbs") or 0.0) / peak_h2d if peak_h2d else None,
        "h2d_expert_gbs": ex.get("h2d_gbs"),
        "host_codec": {"codec": ex.get("host_codec") or "raw", "wire_ratio": ex.get("h2d_wire_ratio")},
        "h2d_expert_bytes_per_step": ex.get("h2d_bytes", 0) / args.steps,
        "h2d_wire_bytes_per_step": ex.get("h2d_wire_bytes", 0) / args.steps,
        "hidden_prefetch_fraction": ex.get("hidden_prefetch_fraction"),
        "stall_ms_per_step": {"prefetch": ex.get("stall_prefetch_ms", 0) / args.steps,
                              "demand": ex.get("stall_demand_ms", 0) / args.steps},
        "roofline_k3": {
            "kernel": "spmoe_expert_ffn_tc_units (K3: unit-fused tcgen05 SwiGLU, both phases per (expert, 128-feature block) + fixed-order partial sum)",
            "bound": "hbm",
            "achieved": roof.get("achieved_gbs"),
            "peak": peaks["hbm_gbs"],
            "peak_source": peaks["source"] + " copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "unit": "GB/s",
            "frac": (roof.get("achieved_gbs") or 0.0) / peaks["hbm_gbs"],
            "traffic": None,
            "launches": roof.get("launches"),
            "ms_per_step": (roof.get("total_ms") or 0.0) / args.steps,
            "bytes_per_launch": roof.get("bytes_per_launch"),
            "ms_per_launch": roof.get("ms_per_launch"),
            "by_shape": roof.get("by_shape"),
            "timing": "device globaltimer span per K3 call (first kernel's first CTA start -> last kernel's last CTA end)",
            "cuda_events": None if not ev_k3 else dict(ev_k3, frac=ev_k3["achieved"] / peaks["hbm_gbs"]),
        },
        # the copy path's XC decode kernel (runs under the copies of later
        # segments; only the last segment of a layer is on the critical path)
        "roofline_decode": None if not dec or not dec["launches"] else {
            "kernel": "xc_decode_kernel (XC blob -> raw expert bf16, one launch per segment)",
            "bound": "hbm", "achieved": dec["gbs"], "peak": peaks["hbm_gbs"],
            "peak_source": peaks["source"] + " copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "unit": "GB/s",
            "frac": (dec["gbs"] or 0.0) / peaks["hbm_gbs"], "traffic": None, "launches": dec["launches"],
            "ms_per_step": dec["ms"] / args.steps,
            "bytes_per_launch": dec["bytes"] / dec["launches"],
            "ms_per_launch": dec["ms"] / dec["launches"],
            "timing": "device globaltimer span per launch (first CTA start -> last CTA end)",
            "cuda_events": None if not ev_dec else dict(ev_dec, frac=ev_dec["achieved"] / peaks["hbm_gbs"]),
        },
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step},
        # Python-issued kernels (K.LAUNCHES) + the runtime's XC decodes
        "gpu_launches": launches + (dec["launches"] if dec else 0),
        "clocks": clk,
    }
    for key, name in (("roofline_k3", "ncu_k3_traffic.json"), ("roofline_decode", "ncu_xc_decode_traffic.json")):
        prof = ROOT / "profiles" / name
        if out.get(key) and prof.exists():
            t = json.loads(prof.read_text())
            out[key]["traffic"] = t.get("traffic_per_launch_bytes")
            out[key]["traffic_source"] = t.get("source")
    # `roofline` = the kernel with the largest GPU time in the timed region
    # (CUDA events around every launch); the other one stays beside it
    cands = [out[k] for k in ("roofline_k3", "roofline_decode") if out.get(k)]
    dom = max(cands, key=lambda r: r["ms_per_step"])
    out["roofline"] = dict(dom, dominant_by="GPU ms per step in the timed region, "
                           + ", ".join(f"{r['kernel'].split(' ')[0]} {r['ms_per_step']:.1f}" for r in cands))
    eng.close()  # releases the pinned host pool before the CPU leg allocates its own weights
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample (~10-30 s of CPU work): full SD iterations of the
        # first CPU_SAMPLE_LAYERS decoder layers of the same model (identical
        # per-layer shapes and arithmetic), time scaled by L / layers; the
        # unscaled full-model loop is `bench.py --impl reference`
        threads = host_threads()
        nl = min(CPU_SAMPLE_LAYERS, arch.num_layers)
        sd, _, _ = cpu_sd(arch, cfg, threads, layers=nl)
        sd.step()  # warm-up
        t0 = time.perf_counter()
        for _ in range(2):
            sd.step()
        t_it = (time.perf_counter() - t0) / 2 * arch.num_layers / nl
        emitted_per_iter = emitted / args.steps
        out["cpu_baseline"] = {
            "value": emitted_per_iter / t_it, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"2 full SD iterations (draft, predictor, verify MoE, lm_head, acceptance) of the first {nl} "
                      f"of {arch.num_layers} layers on oracle/cpu_model.py ({threads} threads), per-layer time "
                      f"scaled to {arch.num_layers} layers; {emitted_per_iter:.2f} tokens/iteration from this "
                      f"GPU run (the unscaled full-model CPU loop is the --impl reference arm)",
            "ms_per_iteration": t_it * 1e3,
        }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
