"""Run records and the metrics contract (drop-in for moesim's SimReport).

``SimReport`` keeps the reference's fields, CSV columns and text summary
(``simcore.py:57-170``); the B200 engine fills it from CUDA-event timelines
instead of a simulated clock and adds measured extras (HBM / H2D bandwidth,
hidden-prefetch fraction, acceptance, routing parity data) in ``extras``.
Transfer and compute-slot CSVs use the reference headers
(``report.py:22-23,45-61``) so moesim's tooling reads B200 timelines.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from pathlib import Path

from .config import PolicySpec


class TransferKind(str, enum.Enum):
    PREFETCH = "prefetch"
    ON_DEMAND = "on_demand"


@dataclass(frozen=True)
class TransferRecord:
    start: float
    end: float
    nbytes: int
    kind: TransferKind
    layer: int
    experts: tuple[int, ...]

    @property
    def duration(self) -> float:
        return self.end - self.start


@dataclass(frozen=True)
class IterationRecord:
    index: int
    start: float
    draft_end: float
    verify_end: float
    position: int
    drafted: int
    accepted: int
    emitted: int


@dataclass(frozen=True)
class ComputeSlot:
    kind: str  # draft | verify
    iteration: int
    token: int
    layer: int
    start: float
    end: float


@dataclass
class SimReport:
    policy: PolicySpec
    seed: int
    tpot: float
    hit_rate: float
    eviction_rate: float
    latency_breakdown: dict[str, float]
    total_time: float
    emitted_tokens: int
    cutoff_effective: int | None
    cache_capacity: int
    iterations: list[IterationRecord]
    transfers: list[TransferRecord]
    compute_slots: list[ComputeSlot]
    counters: dict[str, int]
    extras: dict = field(default_factory=dict)

    CSV_FIELDS = (
        "policy", "seed", "tpot_ms", "hit_rate", "eviction_rate", "frac_draft",
        "frac_expert_load", "frac_attention_other", "total_time_ms", "emitted_tokens",
        "iterations", "cutoff_layer", "cache_capacity", "hits", "misses",
        "prefetch_insertions", "prefetch_evictions", "demand_insertions",
        "tasks_completed", "tasks_aborted",
    )

    @classmethod
    def csv_header(cls) -> str:
        return ",".join(cls.CSV_FIELDS)

    def _values(self) -> dict[str, str]:
        b = self.latency_breakdown
        c = self.counters
        return {
            "policy": self.policy.policy.value,
            "seed": str(self.seed),
            "tpot_ms": f"{self.tpot * 1e3:.3f}",
            "hit_rate": f"{self.hit_rate:.6f}",
            "eviction_rate": f"{self.eviction_rate:.6f}",
            "frac_draft": f"{b['draft']:.6f}",
            "frac_expert_load": f"{b['expert_load']:.6f}",
            "frac_attention_other": f"{b['attention_and_other']:.6f}",
            "total_time_ms": f"{self.total_time * 1e3:.3f}",
            "emitted_tokens": str(self.emitted_tokens),
            "iterations": str(len(self.iterations)),
            "cutoff_layer": "" if self.cutoff_effective is None else str(self.cutoff_effective),
            "cache_capacity": str(self.cache_capacity),
            "hits": str(c["hits"]),
            "misses": str(c["misses"]),
            "prefetch_insertions": str(c["prefetch_insertions"]),
            "prefetch_evictions": str(c["prefetch_evictions"]),
            "demand_insertions": str(c["demand_insertions"]),
            "tasks_completed": str(c["tasks_completed"]),
            "tasks_aborted": str(c["tasks_aborted"]),
        }

    def csv_row(self) -> str:
        v = self._values()
        return ",".join(v[k] for k in self.CSV_FIELDS)

    def to_text(self) -> str:
        b = self.latency_breakdown
        out = [
            f"policy: {self.policy.policy.value}",
            f"seed: {self.seed}",
            f"tpot_ms: {self.tpot * 1e3:.3f}",
            f"total_time_ms: {self.total_time * 1e3:.3f}",
            f"emitted_tokens: {self.emitted_tokens}",
            f"iterations: {len(self.iterations)}",
            f"hit_rate: {self.hit_rate:.6f}",
            f"eviction_rate: {self.eviction_rate:.6f}",
            f"cutoff_layer: {self.cutoff_effective}",
            f"cache_capacity: {self.cache_capacity}",
            "latency_breakdown:",
            f"  draft: {b['draft']:.6f}",
            f"  expert_load: {b['expert_load']:.6f}",
            f"  attention_and_other: {b['attention_and_other']:.6f}",
            "counters:",
        ]
        out += [f"  {k}: {v}" for k, v in sorted(self.counters.items())]
        return "\n".join(out) + "\n"


TRANSFERS_HEADER = "start_ms,end_ms,bytes,kind,layer,expert"
SLOTS_HEADER = "kind,iteration,token,layer,start_ms,end_ms"


def write_transfer_log_csv(report: SimReport, path: str | Path) -> None:
    rows = [TRANSFERS_HEADER]
    for t in report.transfers:
        experts = ";".join(str(e) for e in t.experts)
        rows.append(f"{t.start * 1e3:.3f},{t.end * 1e3:.3f},{t.nbytes},{t.kind.value},{t.layer},{experts}")
    Path(path).write_text("\n".join(rows) + "\n")


def write_compute_slots_csv(report: SimReport, path: str | Path) -> None:
    rows = [SLOTS_HEADER]
    for s in report.compute_slots:
        rows.append(f"{s.kind},{s.iteration},{s.token},{s.layer},{s.start * 1e3:.3f},{s.end * 1e3:.3f}")
    Path(path).write_text("\n".join(rows) + "\n")


def write_report_text(report: SimReport, path: str | Path) -> None:
    Path(path).write_text(report.to_text())


def write_report_csv(reports: list[SimReport], path: str | Path, prefix_cols=()) -> None:
    """One row per report; ``prefix_cols`` = (name, values) leading columns."""
    head = [name for name, _ in prefix_cols] + [SimReport.csv_header()]
    lines = [",".join(head)]
    for i, r in enumerate(reports):
        lines.append(",".join([str(v[i]) for _, v in prefix_cols] + [r.csv_row()]))
    Path(path).write_text("\n".join(lines) + "\n")
