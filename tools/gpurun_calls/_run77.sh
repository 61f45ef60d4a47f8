python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r77_bench_$i.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/r77_bench_$i.log').read().strip().splitlines()[-1]); print('run $i', round(d['value'],1), round(d['e2e']['value'],1), d['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
