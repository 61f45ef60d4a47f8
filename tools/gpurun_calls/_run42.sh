python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r44_build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lz4_decode_map -s 5 -c 1 -o gpurun_out/r2_lz4map3 python tools/bench_ingest.py --bricks 16 > gpurun_out/r44_ncu.log 2>&1
tail -1 gpurun_out/r44_ncu.log
