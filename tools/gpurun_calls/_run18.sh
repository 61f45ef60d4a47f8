python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r18_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ingest.py -q -x > gpurun_out/r18_ingest.log 2>&1; tail -2 gpurun_out/r18_ingest.log
for nb in 1 16 64 4096; do timeout 600 python tools/bench_ingest.py --bricks $nb > gpurun_out/r18_ing_$nb.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r18_ing_$nb.json').read().strip().splitlines()[-1]); print($nb, round(d['gpu_decode_kernel_ms'],3), round(d['gpu_decode_GBps_out'],2), round(d['apply_bricks_lz4_ms'],2))"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_request" > gpurun_out/r18_wide.log 2>&1; tail -3 gpurun_out/r18_wide.log
timeout 900 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_session_api.py -q -x > gpurun_out/r18_abi.log 2>&1; tail -3 gpurun_out/r18_abi.log
