python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r30_build.log 2>&1
python tools/trend_probe.py --mode residency; python tools/trend_probe.py --mode pagetable
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_stats.so python tools/trend_probe.py --mode residency
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_raycast -s 3 -c 1 -o gpurun_out/r2_trend python tools/trend_probe.py --mode residency > gpurun_out/r30_ncu.log 2>&1; tail -1 gpurun_out/r30_ncu.log
