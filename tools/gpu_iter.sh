#!/bin/bash
# One GPU iteration: parity tests (fast subset unless FULL=1), then the bench.
# usage: bash tools/gpu_iter.sh TAG [pytest -k expr]
TAG=${1:-iter}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
if [ "${FULL:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
else
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render_units.py tests/test_gpu_acceptance.py -m gpu -x -q ${2:+-k "$2"} > gpurun_out/${TAG}_pytest.log 2>&1
fi
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.log 2>&1
grep -o '"kernel_ms": {[^}]*}' gpurun_out/${TAG}_bench.log
grep -o '"e2e": {"value": [0-9.]*' gpurun_out/${TAG}_bench.log
