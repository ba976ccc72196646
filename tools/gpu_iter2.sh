# iteration check: sorted-engine + slab + pin tests, then the cfg3 bench line
mkdir -p gpurun_out
export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_gpu_sorted_engine.py tests/test_gpu_slab_engine.py tests/test_gpu_cfg3_pin.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-perf-mode | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['ms_per_step'],4), d.get('stage_ms'), 'frac', round(d['roofline']['frac'],4))"
