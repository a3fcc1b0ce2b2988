"""The replica path of bench.py end to end on one B200: two ranks under
torch.distributed.run (gloo, both on cuda:0 via the SPMOE_BENCH_SHARE_GPU
test hook) on the tiny config — NUMA pool roles, the placement plan
broadcast, the shared /dev/shm XC pool (leader fills, follower attaches),
max-over-ranks timing and the summed token count."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_replicas_share_one_pool():
    env = dict(os.environ, SPMOE_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["tokens_emitted"] >= 2 * 2  # both ranks' streams are summed
    assert line["host_codec"]["codec"] == "xc"
    assert "too small" not in r.stderr  # the tiny pool always fits: the shared path ran


def test_bench_gpus_flag_self_spawns_ranks():
    """`python bench.py --gpus 2` with no torchrun environment launches two
    ranks itself (the driver's SCALE run needs no harness changes) and
    reports n_gpus 2 with both streams' tokens and per-rank link figures."""
    env = dict(os.environ, SPMOE_BENCH_SHARE_GPU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "tiny", "--steps", "2",
           "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["tokens_emitted"] >= 4
    assert len(line["per_rank"]) == 2 and all(p["h2d_peak_gbs"] > 0 for p in line["per_rank"])

