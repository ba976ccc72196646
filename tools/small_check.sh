# cfg0/1/2 benches + warm launch list of cfg1 + the GPU suite
export PYTHONPATH=.
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg0; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/s_$c.json 2>gpurun_out/s_$c.err
  echo "$c rc=$?"; tail -1 gpurun_out/s_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('stage_ms'))"; tail -2 gpurun_out/s_$c.err
done
timeout 600 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/warm_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/warm_cfg1.log 2>&1; echo ncu rc=$?
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -${TEST_TAIL:-15}
