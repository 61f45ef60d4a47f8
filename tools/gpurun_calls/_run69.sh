python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r69_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r69_pytest.log 2>&1; tail -2 gpurun_out/r69_pytest.log
C4_PROFILE_FRAME=9 timeout 900 python tools/bench_config4.py --cold-frames 10 --orbit-frames 1 2>&1 >/dev/null | grep -A14 "^--- apply" | cut -c1-60,100-200
timeout 900 python tools/bench_config4.py > gpurun_out/r69_c4.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r69_c4.json').read().strip().splitlines()[-1]); print('c4', d['frame_ms_excl_fetch'], d['cold']['steady_apply_ms_median'], d['cold']['steady_upload_gbs'], d['cold']['render_ms_median'])"
timeout 900 python tools/bench_config3.py > gpurun_out/r69_c3.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/r69_c3.json').read().strip().splitlines()[-1]); print('c3', d['frame_device_ms'], d['apply_bricks_ms_median'])"
