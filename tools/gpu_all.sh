# whole GPU suite + the small-config bench lines
mkdir -p gpurun_out
export PYTHONPATH=.
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
for c in cfg0 cfg1 cfg2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],5), d.get('stage_ms'), d['gpu_launches'])"
done
