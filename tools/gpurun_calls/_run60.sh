RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_debug.so timeout 900 python -m pytest tests/test_gpu_ingest.py -m gpu -q > gpurun_out/r60_debug_ingest.log 2>&1; tail -2 gpurun_out/r60_debug_ingest.log
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_debug.so timeout 300 python tools/bench_ingest.py --bricks 148 | tail -c 300
timeout 900 python -m pytest tests/test_gpu_ingest.py -m gpu -q > gpurun_out/r60_ingest.log 2>&1; tail -2 gpurun_out/r60_ingest.log
timeout 300 python tools/bench_ingest.py --bricks 16 | tail -c 300
