"""The hot path's kernels first (this file sorts first, so a launch capture
of the GPU suite sees them before the model-building kernels of later
tests): K1 router top-k, K2 permute, K3 on all three paths (unit-fused
tcgen05, two-phase tcgen05, CUDA-core), K4 combine and K6 greedy
acceptance, each against the CPU oracle (the same pass smoke() runs)."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def test_hot_path_kernels_against_oracle(oracle):
    import __graft_entry__ as g

    g._kernel_pass(oracle)
