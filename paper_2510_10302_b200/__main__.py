"""Command line (subset of the reference's ``moesim`` CLI relevant to the path).

  python -m paper_2510_10302_b200 cutoff --config C [--k K] [--side draft|target] [--window N]
      same report as ``moesim cutoff`` (cli.py:197-219), plus the N-token
      drafting-window variant;
  python -m paper_2510_10302_b200 run --config C --arch mixtral_8x7b [--tokens 64] [--out DIR]
      real B200 SD run -> report.txt, report.csv, transfers.csv (reference
      CSV schema), trace.txt (trace-v1 of the real gating scores) and
      profiled.yaml (ProfiledTimings measured on this GPU).

Exit codes follow the reference: 0 ok, 1 validation error, 2 runtime error.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

from .config import ConfigError, ValidationError, load_config
from .cutoff import cutoff_input_from_specs, feasibility_report, solve_cutoff


def cmd_cutoff(a) -> int:
    model, hw, timings, policy = load_config(a.config)
    k = a.k if a.k is not None else policy.prefetch_k
    inp = cutoff_input_from_specs(model, hw, timings, k, side=a.side, window_tokens=a.window)
    res = solve_cutoff(inp)
    print(f"k: {k}")
    print(f"layers considered: 0..{inp.l_all - 1} ({a.side} side)")
    if not res.feasible:
        print("cutoff: none (even layer 0 violates a constraint)")
        print(f"binding constraint: {res.binding_constraint.value}")
        return 0
    fr = feasibility_report(inp, res.layer)
    print(f"cutoff layer L: {res.layer}")
    print(f"prefetched experts n_expert: {res.n_expert}")
    print(f"binding constraint: {res.binding_constraint.value}")
    print(f"memory slack: {fr.memory_slack_bytes / 1e6:.3f} MB")
    print(f"overlap slack: {fr.overlap_slack_seconds * 1000:.3f} ms")
    return 0


def cmd_run(a) -> int:
    import torch

    from .calibrate import measure_timings, write_profiled_config
    from .engine import SpecMoEEngine
    from .model import get_arch, load_arch
    from .report import write_report_csv, write_report_text, write_transfer_log_csv

    model, hw, timings, policy = load_config(a.config)
    arch = load_arch(a.config) or get_arch(a.arch)
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    eng = SpecMoEEngine(arch, hw, timings, policy, batch=1, record_routing=True)
    try:
        g = torch.Generator().manual_seed(policy.seed)
        rep = eng.generate(torch.randint(0, arch.vocab, (1, a.prompt), generator=g), a.tokens)
        write_report_text(rep, out / "report.txt")
        write_report_csv([rep], out / "report.csv")
        write_transfer_log_csv(rep, out / "transfers.csv")
        eng.export_trace(out / "trace.txt")
        write_profiled_config(out / "profiled.yaml", eng.model, eng.effective_hw(), measure_timings(eng), policy)
        print(rep.to_text(), end="")
    finally:
        eng.close()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2510_10302_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("cutoff")
    c.add_argument("--config", required=True)
    c.add_argument("--k", type=int, default=None)
    c.add_argument("--side", choices=["draft", "target"], default="draft")
    c.add_argument("--window", type=int, default=1)
    c.add_argument("--out", default=None)
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--arch", default="tiny")
    r.add_argument("--tokens", type=int, default=64)
    r.add_argument("--prompt", type=int, default=32)
    r.add_argument("--out", default="run_out")
    a = ap.parse_args(argv)
    try:
        return {"cutoff": cmd_cutoff, "run": cmd_run}[a.cmd](a)
    except (ValidationError, ConfigError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except Exception as exc:  # runtime failure
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
