python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r40_build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_lz4_decode_map -s 5 -c 1 -o gpurun_out/r2_lz4map python tools/bench_ingest.py --bricks 16 > gpurun_out/r40_ncu.log 2>&1
tail -2 gpurun_out/r40_ncu.log
