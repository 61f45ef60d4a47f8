python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r70_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_raycast -s 8 -c 1 -o gpurun_out/r2_c4 python tools/bench_config4.py --cold-frames 10 --orbit-frames 1 > gpurun_out/r70_ncu.log 2>&1; tail -1 gpurun_out/r70_ncu.log
