python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r28_build.log 2>&1
timeout 900 python tools/bench_methods.py > gpurun_out/r28_methods96.jsonl 2>&1; tail -4 gpurun_out/r28_methods96.jsonl | cut -c1-400
timeout 900 python tools/bench_methods.py --size 1024 --frames 12 > gpurun_out/r28_methods1024.jsonl 2>&1; tail -4 gpurun_out/r28_methods1024.jsonl | cut -c1-400
timeout 900 python tools/bench_config5.py > gpurun_out/r28_c5.json 2> gpurun_out/r28_c5.err; tail -c 1500 gpurun_out/r28_c5.json
