for v in base eager; do
  L=$PWD/paper_2309_04393_b200/_variants/libresoct_$v.so
  RESOCT_LIB=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r80_$v.log 2>&1
  echo "$v c2 $(grep -o '"raycast": [0-9.]*' gpurun_out/r80_$v.log) trend $(RESOCT_LIB=$L python tools/trend_probe.py --mode residency | grep -o '"kernel_ms": [0-9.]*')"
  RESOCT_LIB=$L timeout 900 python tools/bench_config4.py --cold-frames 10 --orbit-frames 6 > gpurun_out/r80_c4_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r80_c4_$v.json').read().strip().splitlines()[-1]); print('$v c4', d['cold']['render_ms_median'], d['orbit']['render_ms_median'], d['frame_ms_excl_fetch']['p50'])"
done
