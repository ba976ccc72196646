# update-kernel timing under the CS_FAST_DEBUG diagnostics (wrong results)
for d in ${DBG:-0 4 32 36}; do
CS_FAST_DEBUG=$d timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fast_update" -c 3 --csv --log-file gpurun_out/d$d.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "== debug $d"; grep k_fast_update gpurun_out/d$d.csv | tail -3 | cut -d, -f5,13- | cut -c1-200
done
