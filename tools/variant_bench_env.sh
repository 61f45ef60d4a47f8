#!/bin/bash
# like variant_bench.sh, with per-variant environment (sub4 needs 4^3 tables)
mkdir -p gpurun_out
for lib in paper_2309_04393_b200/_variants/libresoct_*.so; do
  name=$(basename $lib .so)
  env=""
  case $name in *sub4*) env="RESOCT_SUB_EDGE_ALLOC=4";; *sub2*) env="RESOCT_SUB_EDGE_ALLOC=2";; esac
  env $env RESOCT_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
     > gpurun_out/var_$name.log 2>&1
  echo "$name $(grep -o '"kernel_ms": {[^}]*}' gpurun_out/var_$name.log)" >> gpurun_out/variants.txt
done
