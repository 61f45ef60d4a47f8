#!/bin/bash
# Round-end evidence on one B200 (every command after the build must first
# exit 0 on its own; ncu runs only after the plain run of the same command).
# usage: bash tools/gpu_final.sh TAG   -> gpurun_out/TAG_*
T=${1:-final}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; tail -1 $O/${T}_pytest_gpu.log
timeout 900 python bench.py > $O/${T}_bench.log 2>&1; echo "bench rc=$?"; tail -c 600 $O/${T}_bench.log
timeout 900 python bench.py --impl reference > $O/${T}_bench_reference.log 2>&1; echo "reference rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/${T}_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_raycast -s 3 -c 1 \
  -o $O/${T}_raycast python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/${T}_raycast_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/bench_config5.py > $O/${T}_c5.json 2> $O/${T}_c5.err; echo "c5 rc=$?"
timeout 900 python tools/bench_methods.py > $O/${T}_methods96.jsonl 2>&1; echo "m96 rc=$?"
timeout 900 python tools/bench_methods.py --size 1024 --frames 12 > $O/${T}_methods1024.jsonl 2>&1; echo "m1024 rc=$?"
timeout 900 python tools/bench_config3.py > $O/${T}_c3.json 2> $O/${T}_c3.err; echo "c3 rc=$?"
timeout 1200 python tools/bench_config4.py > $O/${T}_c4.json 2> $O/${T}_c4.err; echo "c4 rc=$?"
for n in 16 148 4096; do timeout 300 python tools/bench_ingest.py --bricks $n > $O/${T}_ingest_$n.json 2>&1; done; echo ingest done
