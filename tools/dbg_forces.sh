# force-kernel timing under the CS_FAST_DEBUG diagnostics (wrong results)
for d in 0 64 128; do
CS_FAST_DEBUG=$d timeout 200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_fast_forces" -c 3 --csv --log-file gpurun_out/fd$d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "== debug $d"; grep k_fast_forces gpurun_out/fd$d.csv | tail -2 | cut -d, -f13- | cut -c1-150
done
