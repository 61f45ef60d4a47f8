python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r32_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render_units.py tests/test_gpu_acceptance.py -m gpu -x -q > gpurun_out/r32_pytest.log 2>&1; tail -2 gpurun_out/r32_pytest.log
for v in base new; do
  if [ $v = new ]; then L=$PWD/paper_2309_04393_b200/libresoct.so; else L=$PWD/paper_2309_04393_b200/_variants/libresoct_base.so; fi
  RESOCT_LIB=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r32_bench_$v.log 2>&1
  echo "$v $(grep -o '"kernel_ms": {[^}]*}' gpurun_out/r32_bench_$v.log) $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/r32_bench_$v.log)"
  RESOCT_LIB=$L python tools/trend_probe.py --mode residency
done
python tools/trend_probe.py --mode pagetable
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"classify|k_raycast" -c 6 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "k_classify|k_raycast|gpu__time" | head -12
