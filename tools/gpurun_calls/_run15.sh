FULL=1 bash tools/gpu_iter.sh it15
python tools/first_frame.py > gpurun_out/r15_ff.log 2>&1; tail -c 600 gpurun_out/r15_ff.log; echo
timeout 900 python tools/bench_config3.py > gpurun_out/r15_c3.json 2> gpurun_out/r15_c3.err; python -c "
import json; d=json.load(open('gpurun_out/r15_c3.json')); print({k: d[k] for k in ('frame_device_ms','render_ms','apply_bricks_ms_median','render_ms_median')})"
timeout 1200 python tools/bench_config4.py --cold-frames 20 --orbit-frames 12 > gpurun_out/r15_c4.json 2> gpurun_out/r15_c4.err; python -c "
import json; d=json.load(open('gpurun_out/r15_c4.json')); print({k: d[k] for k in ('first_frames_ms','frame_ms_excl_fetch','reserve_s','setup_s')}); print(d['orbit'])"
