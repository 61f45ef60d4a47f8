python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b3_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_feedback.py -x -q > gpurun_out/b3_fb.log 2>&1; tail -15 gpurun_out/b3_fb.log
FULL=1 bash tools/gpu_iter.sh full3
