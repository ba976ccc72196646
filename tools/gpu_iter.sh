# iteration check: sorted-engine GPU tests, bench (no baselines), launch list,
# and an ncu --set full capture of the kernels named in $NCU_K (optional)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_sorted_engine.py -q -x 2>&1 | tail -3
timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err; tail -2 gpurun_out/b.err
head -c 330 gpurun_out/b.json; echo
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1
if [ -n "$NCU_K" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" --launch-skip ${NCU_SKIP:-4} -c ${NCU_C:-2} -o gpurun_out/full_it -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_f.log 2>&1; echo ncu $?
fi
