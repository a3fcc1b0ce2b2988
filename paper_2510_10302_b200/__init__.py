"""B200-native SP-MoE verification-time expert path.

Drop-in for the reference package ``moesim`` (arxiv 2510.10302) on the path
named by BASELINE.json: model/config loading, the draft/target SD loop, the
prefetch-policy and cutoff-layer knobs keep the reference names and
semantics; the arithmetic runs in hand-written sm_100a kernels behind the C
ABI of ``include/spmoe.h`` (``libspmoe.so``), with no CPU fallback.

Importing this package does not touch CUDA; the native library is loaded on
first use (:mod:`._native`).
"""

from .cache import CacheError, ExpertCache, ExpertId, InsertKind, NativeExpertCache
from .config import (
    ConfigError,
    HardwareSpec,
    ModelSpec,
    Policy,
    PolicySpec,
    ProfiledTimings,
    ValidationError,
    cache_capacity_slots,
    derive_expert_io_time,
    load_config,
    parse_bytes,
    specs_from_dict,
    validate_timings,
    with_policy,
    write_config,
)
from .cutoff import (
    BindingConstraint,
    CutoffInput,
    CutoffResult,
    FeasibilityReport,
    cutoff_input_from_specs,
    feasibility_report,
    solve_cutoff,
)
from .predictor import CriticalExpertSet, DraftGuidedPredictor, HistoryCounter, select_critical, top_k_indices
from .report import (
    ComputeSlot,
    IterationRecord,
    SimReport,
    TransferKind,
    TransferRecord,
    write_compute_slots_csv,
    write_report_csv,
    write_report_text,
    write_transfer_log_csv,
)

__version__ = "0.1.0"


def __getattr__(name):
    # engine / model pull in torch CUDA state; import lazily
    if name in ("SpecMoEEngine", "simulate", "effective_cutoff", "compare_policies", "sweep",
                "SWEEP_PARAMETERS"):
        from . import engine

        return getattr(engine, name)
    if name in ("ArchSpec", "ARCH_PRESETS", "get_arch", "load_arch", "model_spec_for"):
        from . import model

        return getattr(model, name)
    raise AttributeError(name)
