#!/bin/bash
# GPU round: full GPU suite (no -x), two bench runs (reproducibility), smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/gt.log 2>&1
tail -5 gpurun_out/gt.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python - <<'PY'
import json
for f in ("gpurun_out/bench.json", "gpurun_out/bench2.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["acceptance_rate"], d["tokens_emitted"], d["roofline"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
echo done
