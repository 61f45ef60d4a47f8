python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r43_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_ingest.py -m gpu -x -q 2>&1 | tail -3
for L in paper_2309_04393_b200/libresoct.so paper_2309_04393_b200/_variants/libresoct_pipe.so; do
  echo "== $L"
  for n in 1 16 64 148 4096; do
    RESOCT_LIB=$PWD/$L timeout 300 python tools/bench_ingest.py --bricks $n | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($n, round(d['gpu_decode_kernel_ms'],3), round(d['gpu_decode_GBps_out'],2), round(d['apply_bricks_lz4_ms'],2))"
  done
done
