rm -f gpurun_out/variants.txt
for lib in paper_2309_04393_b200/_variants/libresoct_*.so; do
  name=$(basename $lib .so)
  for rep in 1 2; do
  RESOCT_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_$name.log 2>&1
  echo "$name $(grep -o '"kernel_ms": {[^}]*}' gpurun_out/var_$name.log) trend $(RESOCT_LIB=$PWD/$lib python tools/trend_probe.py --mode residency | grep -o '"kernel_ms": [0-9.]*')" >> gpurun_out/variants.txt
  done
done
cat gpurun_out/variants.txt
