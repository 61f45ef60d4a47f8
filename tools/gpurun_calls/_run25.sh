python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r25_build.log 2>&1
timeout 600 python tools/profile_apply.py 55 > gpurun_out/r25_apply.log 2>&1; cat gpurun_out/r25_apply.log | grep -v Warning | head -60
