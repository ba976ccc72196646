# Round measurement set: GPU tests, full bench, reference arm, launch list,
# one ncu --set full capture of the force/update/sort kernels (after the same
# command has exited 0 without ncu).
mkdir -p gpurun_out
set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/ref.err; echo ref rc=$?
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.json 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fast_forces|k_fast_update|k_scan|k_bucket_sort|k_fast_deposit_rows|k_spec_cols" --launch-skip 12 -c 7 -o gpurun_out/full_cfg3 -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f.log 2>&1; echo ncu2 rc=$?
