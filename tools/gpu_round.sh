#!/bin/bash
# One GPU round (run under gpurun from the repo root):
#   build, full -m gpu suite, bench (XC tier, headline) + raw tier + reference
#   arm, launch list of one bench iteration (ncu, --cutoff 1 so the
#   recalibration under the profiler does not move the cutoff), smoke.
# Outputs land in gpurun_out/ (bench_xc.json, bench_raw.json, bench_ref.json,
# launches_xc.csv, gt.log, ...).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/gt.log 2>&1; tail -3 gpurun_out/gt.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_xc.json 2> gpurun_out/bench_xc.err
timeout 900 python bench.py --steps 20 --warmup 3 --host-codec none --no-cpu-baseline > gpurun_out/bench_raw.json 2> gpurun_out/bench_raw.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_xc.json", "gpurun_out/bench_raw.json", "gpurun_out/bench_ref.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k: d.get(k) for k in ("value", "tpot_ms", "acceptance_rate", "h2d_gbs", "h2d_expert_gbs", "ms_per_step", "cutoff_layer")},
              (d.get("roofline") or {}).get("frac"), (d.get("roofline_decode") or {}).get("frac"),
              (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
SPMOE_PROFILE_RANGE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_xc.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --cutoff 1 > gpurun_out/bench_ncu.json 2> gpurun_out/bench_ncu.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
echo done
