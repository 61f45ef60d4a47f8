python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r59_build.log 2>&1
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_debug.so RESOCT_FUZZ_N=200 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r59_debug_suite.log 2>&1; tail -2 gpurun_out/r59_debug_suite.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_ingest.py -m gpu -q -x -k "lz4" > gpurun_out/r59_memcheck_lz4.log 2>&1; tail -4 gpurun_out/r59_memcheck_lz4.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "path_class or partial_residency or golden" > gpurun_out/r59_memcheck_parity.log 2>&1; tail -4 gpurun_out/r59_memcheck_parity.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/bench_ingest.py --bricks 16 > gpurun_out/r59_racecheck_lz4.log 2>&1; tail -4 gpurun_out/r59_racecheck_lz4.log
