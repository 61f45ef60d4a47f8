python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r73_bench.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r73_bench.log').read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['clocks'])"
timeout 900 python tools/bench_config3.py > gpurun_out/r73_c3.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r73_c3.json').read().strip().splitlines()[-1]); print('c3', d['frame_device_ms'], d['render_ms_median'])"
