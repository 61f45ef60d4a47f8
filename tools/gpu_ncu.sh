#!/bin/bash
# ncu --set full capture of the ray cast (and optionally the feedback kernel)
# at config 2, after a plain run of the same command exited 0.
# usage: bash tools/gpu_ncu.sh TAG [kernel-regex]
TAG=${1:-ncu}
K=${2:-k_raycast}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 3 -c 1 \
  -o gpurun_out/${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
