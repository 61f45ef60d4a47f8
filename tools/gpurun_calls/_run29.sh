python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r29_build.log 2>&1
timeout 600 python tools/profile_apply.py 55 > gpurun_out/r29_apply.log 2>&1; grep -E "^---|k_octree|k_sub_max" gpurun_out/r29_apply.log | cut -c1-60,150-175
FULL=1 bash tools/gpu_iter.sh it29
