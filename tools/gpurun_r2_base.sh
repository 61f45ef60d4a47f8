set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2_base.log 2>&1
tail -c 3000 gpurun_out/bench_r2_base.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_raycast -s 3 -c 1 -o gpurun_out/r2_base_raycast python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_base.log 2>&1
tail -5 gpurun_out/ncu_base.log
