# quick GPU check: big-N sanity, GPU test suite, bench, launch list
mkdir -p gpurun_out
export PYTHONPATH=.
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/run_steps.py 10000000 3 2>&1 | grep -E "step|Error" | head -4
timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err; tail -2 gpurun_out/b.err
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1
