"""The package façade: every name the lazy export list advertises resolves,
and ``sweep`` / ``compare_policies`` keep the reference's signature and
validation rules (``simcore.py:518-564``); on the GPU they run the real
engine over one shared model build."""

from __future__ import annotations

import pytest

import paper_2510_10302_b200 as m
from paper_2510_10302_b200 import HardwareSpec, Policy, PolicySpec, ProfiledTimings, ValidationError


def specs(policy=Policy.DRAFT_PREFETCH, cutoff=2):
    from paper_2510_10302_b200.model import get_arch, model_spec_for

    a = get_arch("tiny")
    hw = HardwareSpec(gpu_memory=180_000_000_000, peak_non_expert_memory=8_000_000_000, pcie_bandwidth=55e9)
    t = ProfiledTimings(t_comp_target=1e-4, t_comp_draft=1e-4, t_io_expert=a.expert_bytes / 55e9)
    pol = PolicySpec(policy=policy, prefetch_k=1, draft_length=4, acceptance_rate=1.0, seed=1234,
                     cutoff_layer=cutoff if policy is Policy.DRAFT_PREFETCH else None, cache_capacity_experts=12)
    return model_spec_for(a), hw, t, pol, a


def test_lazy_exports_resolve():
    for name in ("SpecMoEEngine", "simulate", "effective_cutoff", "compare_policies", "sweep", "SWEEP_PARAMETERS",
                 "ArchSpec", "ARCH_PRESETS", "get_arch", "load_arch", "model_spec_for"):
        assert getattr(m, name) is not None, name
    with pytest.raises(AttributeError):
        m.not_a_name  # noqa: B018


def test_sweep_parameters_match_reference():
    assert m.SWEEP_PARAMETERS == {
        "cutoff_layer": "cutoff_layer",
        "draft_length": "draft_length",
        "cache_capacity": "cache_capacity_experts",
        "prefetch_k": "prefetch_k",
    }


def test_sweep_validation_like_reference():
    model, hw, t, pol, a = specs()
    with pytest.raises(ValidationError, match="unknown sweep parameter"):
        m.sweep("bogus", [1], model, hw, t, pol, arch=a)
    with pytest.raises(ValidationError, match="sweep range is empty"):
        m.sweep("cutoff_layer", [], model, hw, t, pol, arch=a)
    _, _, _, od, _ = specs(Policy.ON_DEMAND)
    with pytest.raises(ValidationError, match="require the draft_prefetch"):
        m.sweep("cutoff_layer", [1], model, hw, t, od, arch=a)
    with pytest.raises(ValidationError, match="does not apply to the on_demand"):
        m.sweep("prefetch_k", [1], model, hw, t, od, arch=a)
    with pytest.raises(ValidationError, match="hidden states"):
        m.sweep("draft_length", [2], model, hw, t, pol, trace=object(), arch=a)
    assert m.compare_policies(model, hw, t, [], arch=a) == []


@pytest.mark.gpu
def test_sweep_and_compare_policies_run_real_engine():
    model, hw, t, pol, a = specs()
    res = m.sweep("cutoff_layer", [0, 3], model, hw, t, pol, arch=a, max_new_tokens=10)
    assert [v for v, _ in res] == [0, 3]
    for v, rep in res:
        assert rep.cutoff_effective == v
        assert sum(it.emitted for it in rep.iterations) >= 10
    res = m.sweep("draft_length", [2, 4], model, hw, t, pol, arch=a, max_new_tokens=10)
    assert [r.iterations[0].drafted for _, r in res] == [2, 4]
    _, _, _, od, _ = specs(Policy.ON_DEMAND)
    reps = m.compare_policies(model, hw, t, [pol, od], arch=a, max_new_tokens=10)
    assert len(reps) == 2
    assert reps[1].counters["prefetch_insertions"] == 0
    # identical model and prompts: greedy decoding emits the same tokens
    # whatever the policy, so the totals agree
    assert sum(i.emitted for i in reps[0].iterations) == sum(i.emitted for i in reps[1].iterations)
