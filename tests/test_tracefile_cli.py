"""CPU tests of the §8(f) output rows: trace-v1 export readable by the
reference's own ``moesim.load_trace`` (when present), ProfiledTimings YAML
round trip, and the ``cutoff`` CLI matching the reference's report."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2510_10302_b200.__main__ import main
from paper_2510_10302_b200.tracefile import read_trace, softmax_rows, write_trace

REF_SRC = Path("/root/reference/pkg/src")
REF_CFG = Path("/root/reference/pkg/configs")


def test_trace_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    scores = softmax_rows(rng.standard_normal((7, 4, 8)))
    write_trace(tmp_path / "t.txt", scores, "tiny", 2, 0, 1234)
    fields, back = read_trace(tmp_path / "t.txt")
    assert fields["layers"] == "4" and fields["experts"] == "8" and fields["topk"] == "2"
    assert np.allclose(back, scores)


def test_trace_loads_in_reference_moesim(tmp_path):
    if not REF_SRC.exists():
        pytest.skip("reference not present")
    sys.path.insert(0, str(REF_SRC))
    try:
        import moesim.trace as mt
    finally:
        sys.path.remove(str(REF_SRC))
    rng = np.random.default_rng(1)
    scores = softmax_rows(rng.standard_normal((5, 3, 8)) * 3)
    write_trace(tmp_path / "t.txt", scores, "tiny", 2, 0, 7)
    tr = mt.load_trace(tmp_path / "t.txt")
    assert tr.num_tokens == 5 and tr.num_layers == 3 and tr.experts_per_layer == 8
    for t in range(5):
        for l in range(3):
            want = tuple(int(i) for i in np.lexsort((np.arange(8), -scores[t, l]))[:2])
            assert tr.layer(t, l).activated == want


def test_profiled_yaml_roundtrip(tmp_path):
    from paper_2510_10302_b200 import HardwareSpec, ModelSpec, Policy, PolicySpec, ProfiledTimings, load_config
    from paper_2510_10302_b200.calibrate import write_profiled_config

    m = ModelSpec("mixtral_8x7b", 32, 8, 2, 0, 352321536, 32)
    h = HardwareSpec(192_000_000_000, 24_000_000_000, 55.5e9, name="b200")
    t = ProfiledTimings(0.0011, 0.00019, 352321536 / 55.5e9 + 2e-5, 2.5e-5)
    p = PolicySpec(Policy.DRAFT_PREFETCH, 1, 4, 1.0, 1234, cache_capacity_experts=64)
    write_profiled_config(tmp_path / "p.yaml", m, h, t, p)
    m2, h2, t2, p2 = load_config(tmp_path / "p.yaml")
    assert (m2, h2, p2) == (m, h, p)
    assert t2.t_io_expert == pytest.approx(t.t_io_expert) and t2.t_comp_draft == pytest.approx(t.t_comp_draft)


def test_cutoff_cli_matches_reference_report(capsys):
    if not REF_CFG.exists():
        pytest.skip("reference configs not present")
    assert main(["cutoff", "--config", str(REF_CFG / "mixtral_measured.yaml")]) == 0
    out = capsys.readouterr().out
    assert "cutoff layer L: 5" in out and "n_expert: 6" in out and "binding constraint: overlap" in out
    assert main(["cutoff", "--config", str(REF_CFG / "mixtral_measured.yaml"), "--window", "4"]) == 0
    assert "cutoff layer L:" in capsys.readouterr().out


def test_cli_exit_codes(tmp_path, capsys):
    bad = tmp_path / "bad.yaml"
    bad.write_text("model: {name: x}\n")
    assert main(["cutoff", "--config", str(bad)]) == 1
