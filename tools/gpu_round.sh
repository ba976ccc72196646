mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench.err; echo bench rc=$?
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_fast_forces|k_fast_update|k_scan|k_fast_scatter" --launch-skip 8 -c 4 -o gpurun_out/full_cfg3 -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f.log 2>&1; echo ncu2 rc=$?
