bash tools/gpu_iter.sh it9
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config2_full_frame" > gpurun_out/r9_full.log 2>&1; tail -2 gpurun_out/r9_full.log
bash tools/gpu_ncu.sh r2_it9
