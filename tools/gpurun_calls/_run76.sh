RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_wtiles.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render_units.py tests/test_gpu_acceptance.py -m gpu -x -q > gpurun_out/r76_pytest.log 2>&1; tail -2 gpurun_out/r76_pytest.log
bash tools/gpurun_calls/_run33.sh
for v in base wtiles; do
  RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_$v.so timeout 900 python tools/bench_config4.py --cold-frames 10 --orbit-frames 6 > gpurun_out/r76_c4_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r76_c4_$v.json').read().strip().splitlines()[-1]); print('$v c4', d['cold']['render_ms_median'], d['orbit']['render_ms_median'], d['frame_ms_excl_fetch']['p50'])"
  RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_$v.so timeout 600 python tools/bench_config5.py --frames 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5', d['frames_per_s'])"
done
