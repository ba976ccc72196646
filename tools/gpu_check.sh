# GPU check after a change: selected GPU tests ($TESTS, default all), then
# short benches of the configs in $CFGS (no baselines), stage times included.
mkdir -p gpurun_out
export PYTHONPATH=.
timeout ${TEST_TIMEOUT:-900} python -m pytest ${TESTS:-tests} -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -${TEST_TAIL:-15}
for c in ${CFGS:-cfg3}; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  echo "== $c rc=$?"; python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/b_{c}.json").read().strip().splitlines()[-1])
    print(c, "ms/step", round(d["ms_per_step"], 4), "value %.3e" % d["value"], "stages", d.get("stage_ms"))
except Exception as e:
    print(c, "no result", e, open(f"gpurun_out/b_{c}.err").read()[-800:])
PY
done
