# Force-kernel queue depth sweep (DESIGN 6a): bench line, kernel time, L1 / L2 hit rates,
# resident warps and instruction count of k_fast_forces / k_fast_forces_generic for the default
# build and the CS_ACC_MAX = 6 / 4 variants.  Build the variants first (here, no GPU needed):
#   python -c "from paper_1805_11007_b200 import build as b; \
#     [b.build(out=f'paper_1805_11007_b200/_build/var/acc{k}.so', extra=[f'-DCS_ACC_MAX={k}']) for k in (6, 4)]"
export PYTHONPATH=.
mkdir -p gpurun_out/s5
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for v in base acc6 acc4; do
  if [ "$v" = base ]; then L=""; else L="paper_1805_11007_b200/_build/var/$v.so"; fi
  CS_LIB=$L timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-perf-mode > gpurun_out/s5/sw_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/s5/sw_$v.json'));print('$v',d['ms_per_step'],d['stage_ms'])"
  CS_LIB=$L timeout 300 ncu --metrics $M --clock-control none -k regex:"k_fast_forces" --launch-skip 6 -c 4 --csv --log-file gpurun_out/s5/sw_$v.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-perf-mode > /dev/null 2>&1
  python - <<P
import csv
rows=[r for r in csv.reader(open('gpurun_out/s5/sw_$v.csv')) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r))
    print('  ',d['Kernel Name'][:40],d['Metric Name'],d['Metric Value'])
P
done
