# Round measurement set (round 2): GPU tests, the default bench (cfg3, with
# the end-to-end, perf-mode and CPU-baseline legs), the reference arm, the
# other configs, the fig1 ensemble, the periodic-solve comparison, the ncu
# launch list of cfg3, one ncu --set full capture of the step's kernels,
# FP64 instruction counts of the cfg2 force kernel, and the update kernel's
# atomics.  Each ncu command runs after the same command exited 0 without it.
set -x
O=gpurun_out/r02
mkdir -p $O
export PYTHONPATH=.
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_reference_cfg3.json 2> $O/ref.err; echo ref rc=$?
for c in cfg0 cfg1 cfg2 cfg2f32 cfg4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo $c rc=$?
done
# the small configs over their whole 1000-step workload (one call: launch overhead amortised)
for c in cfg0 cfg1; do
  timeout 900 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline > $O/bench_${c}_1000steps.json 2> $O/bench_${c}_1000.err; echo $c-1000 rc=$?
done
timeout 900 python bench_ensemble.py > $O/bench_ensemble_fig1.json 2> $O/ens.err; echo ens rc=$?
timeout 600 python tools/spec_bench.py > $O/spec_bench.txt 2>&1; echo spec rc=$?
A="bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-perf-mode"
timeout 300 python $A > $O/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg3.csv python $A > $O/ncu_l.log 2>&1; echo ncu1 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fast_forces|k_fast_update|k_bucket_sort|k_fast_deposit_rows|k_spec_|k_gradient|k_scan" --launch-skip 14 -c 10 -o $O/full_cfg3 -f python $A > $O/ncu_f.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --metrics lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fast_update|k_bucket_sort" -c 4 --launch-skip 2 --csv --log-file $O/atomics_update.csv python $A > $O/ncu_a.log 2>&1; echo ncu3 rc=$?
B="bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 python $B > $O/plain2.json 2>&1 && \
timeout 900 ncu --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,gpu__time_duration.sum --clock-control none -k regex:"k_soft_forces" -c 3 --launch-skip 2 --csv --log-file $O/fp64_cfg2.csv python $B > $O/ncu_fp64.log 2>&1; echo ncu4 rc=$?
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_peak tools/microbench/fp64_peak.cu && /tmp/fp64_peak > $O/fp64_peak.json; cat $O/fp64_peak.json
