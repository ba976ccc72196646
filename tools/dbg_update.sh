for d in 0 4 8 1; do
CS_FAST_DEBUG=$d timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fast_update" -c 3 --csv --log-file gpurun_out/d$d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "== debug $d"; python tools/launches.py gpurun_out/d$d.csv
done
