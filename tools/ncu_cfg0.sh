export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 ncu --set full --sampling-interval 0 --clock-control none --import-source on -k regex:"k_ensemble" --launch-skip 1 -c 1 -o gpurun_out/full_cfg0 -f python bench.py --config cfg0 --steps 1000 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c0.log 2>&1; echo ncu $?
