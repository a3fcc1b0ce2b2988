mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 0 1 0 1; do
SPMOE_XC_STCS=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-event-pass > gpurun_out/ab_$v.json 2>/dev/null
python - $v <<'PY'
import json,sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
k=d["roofline_k3"]; dd=d["roofline_decode"]
print("stcs", sys.argv[1], "ms/step %.1f" % d["ms_per_step"], "k3 frac %.3f" % k["frac"], "1x1", k["by_shape"].get("1x1"), "1x2", k["by_shape"].get("1x2"), "5x9", k["by_shape"].get("5x9"), "decode frac %.3f us %.1f" % (dd["frac"], dd["ms_per_launch"]*1e3))
PY
done
