# after the CTA / ensemble kernel change: whole GPU suite, cfg0 / cfg1 lines, the fig1 ensemble
mkdir -p gpurun_out/r02
export PYTHONPATH=.
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02/gpu_tests.log 2>&1; tail -2 gpurun_out/r02/gpu_tests.log
for c in cfg0 cfg1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err; echo $c rc=$?
done
timeout 900 python bench_ensemble.py > gpurun_out/r02/bench_ensemble_fig1.json 2> gpurun_out/r02/ens.err; echo ens rc=$?
