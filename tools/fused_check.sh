export PYTHONPATH=.
mkdir -p gpurun_out
for F in 0 1; do
  CS_FUSED=$F timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-perf-mode > gpurun_out/fz_$F.json 2>gpurun_out/fz_$F.err
  echo "fused=$F rc=$?"; tail -1 gpurun_out/fz_$F.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('stage_ms'), d['roofline'])"
  tail -3 gpurun_out/fz_$F.err
done
CS_FUSED=1 timeout 900 python -m pytest tests/test_gpu_sorted_engine.py tests/test_gpu_cfg3_pin.py tests/test_gpu_slab_engine.py tests/test_gpu_t4.py -m gpu -q -x 2>&1 | tail -8
