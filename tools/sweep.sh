# Tuning sweep: for each alternative build under _build/var, the bench step
# time and the launch times of the named kernels.  usage: sweep.sh REGEX [names...]
mkdir -p gpurun_out
RX=$1; shift
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="paper_1805_11007_b200/_build/var/$v.so"; fi
  ms=$(CS_LIB=$L timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  CS_LIB=$L timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$RX" -c 6 --csv --log-file gpurun_out/sw_$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  t=$(CS_LIB=$L timeout 300 python -m pytest tests/test_gpu_sorted_engine.py tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -1)
  echo "== $v ms/step=$ms [$t]"; python tools/launches.py gpurun_out/sw_$v.csv
done
