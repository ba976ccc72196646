# ncu --set full of one cfg3 step's F+U kernels (forces, generic pass, update, bucket sort), source-correlated
mkdir -p gpurun_out
export PYTHONPATH=.
A="bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-perf-mode"
timeout 300 python $A > gpurun_out/plain.json 2>gpurun_out/plain.err && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fast_forces|k_fast_update|k_bucket_sort" --launch-skip 8 -c 4 -o gpurun_out/full_fu -f python $A > gpurun_out/ncu_fu.log 2>&1; echo ncu $?
