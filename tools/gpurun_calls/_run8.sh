python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r8_build.log 2>&1
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_stats.so python tools/kernel_stats.py 4 > gpurun_out/r8_stats.log 2>&1
cat gpurun_out/r8_stats.log | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config2_full_frame" > gpurun_out/r8_full.log 2>&1; tail -3 gpurun_out/r8_full.log
bash tools/gpu_ncu.sh r2_it8
