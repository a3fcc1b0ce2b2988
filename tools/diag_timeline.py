"""Per-layer timeline of one Mixtral SD iteration (raw vs XC host tier):
for every verify layer, when its demand copies start, when the last H2D
lands, when its last expert is decoded/usable, when the layer's compute
slot ends and when the next layer's copies start (the link's idle gap)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec
from paper_2510_10302_b200.calibrate import b200_timings
from paper_2510_10302_b200.engine import SpecMoEEngine
from paper_2510_10302_b200.model import get_arch


def run(codec, state=None):
    arch = get_arch("mixtral_8x7b")
    hw = HardwareSpec(gpu_memory=183_359 * 2**20, peak_non_expert_memory=24 * 10**9, pcie_bandwidth=55.5e9,
                      name="b200")
    pol = PolicySpec(policy=Policy.DRAFT_PREFETCH, prefetch_k=1, draft_length=4, acceptance_rate=1.0, seed=1234,
                     cache_capacity_experts=64)
    eng = SpecMoEEngine(arch, hw, b200_timings(arch, hw), pol, batch=1, max_tokens=64 + 64 * 5, window_tokens=4,
                        record_timeline=True, host_codec=codec)
    g = torch.Generator().manual_seed(1000)
    eng.prefill(torch.randint(0, arch.vocab, (1, 64), generator=g))
    for _ in range(3):
        eng.step()
    torch.cuda.synchronize()
    eng._reset_run_state()
    eng.cache.clear_log()
    eng.step()
    torch.cuda.synchronize()
    rep = eng.report()
    log = eng.cache.transfer_log()
    slots = [(s.kind, s.layer, s.start * 1e3, s.end * 1e3) for s in rep.compute_slots]
    t0 = min([r["start_ms"] for r in log] + [s[2] for s in slots])
    rows = []
    vs = {s[1]: s for s in slots if s[0] == "verify"}
    routes = {l: eng.cache.since_epoch_ms(ev) for it, l, ev in eng.route_events}
    dem = {r["layer"]: r for r in log if r["kind"] == "on_demand"}
    for l in range(arch.num_layers):
        r, s = dem.get(l), vs.get(l)
        nxt = dem.get(l + 1)
        rows.append({
            "l": l, "n": r["n_experts"] if r else 0,
            "slot": [round(s[2] - t0, 2), round(s[3] - t0, 2)] if s else None,
            "copy": [round(r["start_ms"] - t0, 2), round(r["copy_end_ms"] - t0, 2), round(r["end_ms"] - t0, 2)] if r else None,
            "gap_to_next_copy": round(nxt["start_ms"] - r["copy_end_ms"], 3) if (r and nxt) else None,
            # pre-MoE block of this layer (slot start -> routing known) and the
            # host's reaction (routing known -> first copy of the layer issued)
            "pre_moe_ms": round(routes[l] - (s[2]), 3) if (s and l in routes) else None,
            "host_ms": round(r["start_ms"] - routes[l], 3) if (r and l in routes) else None,
        })
    ex = rep.extras
    print(json.dumps({"codec": codec, "device_ms": ex["device_ms"], "link_busy_ms": ex["link_busy_ms"],
                      "wire_gbs": ex["h2d_wire_gbs"], "draft_slots": [(round(s[2] - t0, 2), round(s[3] - t0, 2)) for s in slots if s[0] == "draft"],
                      "prefetch": [(r["layer"], r["n_experts"], round(r["start_ms"] - t0, 2), round(r["copy_end_ms"] - t0, 2)) for r in log if r["kind"] == "prefetch"]}), flush=True)
    for row in rows:
        print(json.dumps(row), flush=True)
    eng.close()
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for c in sys.argv[1:] or ["xc", "none"]:
        run(None if c == "none" else c)
