python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r26_build.log 2>&1
timeout 600 python tools/profile_apply.py 55 > gpurun_out/r26_apply.log 2>&1; grep -E "^---|k_|Memcpy" gpurun_out/r26_apply.log | cut -c1-60,150-175
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_state_api.py tests/test_gpu_octree_api.py -q -x -k "lru or octree or session or sub_block or procedural or config3 or swap" > gpurun_out/r26_tests.log 2>&1; tail -2 gpurun_out/r26_tests.log
timeout 900 python tools/bench_config3.py > gpurun_out/r26_c3.json 2> gpurun_out/r26_c3.err; python -c "
import json; d=json.load(open('gpurun_out/r26_c3.json')); print({k: d[k] for k in ('frame_device_ms','render_ms','apply_bricks_ms_median','apply_bricks_us_per_brick_median')})"
