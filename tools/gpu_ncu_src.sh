# ncu --set full, source-correlated, of one launch each of the cfg3 step's issue-bound kernels
mkdir -p gpurun_out/s5
export PYTHONPATH=.
A="bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-perf-mode"
timeout 300 python $A > gpurun_out/s5/plain.json 2>gpurun_out/s5/plain.err && \
for k in k_bucket_sort k_fast_update k_fast_deposit_rows k_fast_forces; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k\$" --launch-skip 3 -c 1 -o gpurun_out/s5/src_$k -f python $A > gpurun_out/s5/ncu_$k.log 2>&1; echo $k ncu $?
done
ls -la gpurun_out/s5/*.ncu-rep
