python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r20_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ingest.py -q -x > gpurun_out/r20_ingest.log 2>&1; tail -2 gpurun_out/r20_ingest.log
for nb in 1 16 64 4096; do timeout 600 python tools/bench_ingest.py --bricks $nb > gpurun_out/r20_ing_$nb.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r20_ing_$nb.json').read().strip().splitlines()[-1]); print($nb, round(d['gpu_decode_kernel_ms'],3), round(d['gpu_decode_GBps_out'],2), round(d['apply_bricks_lz4_ms'],2))"; done
