RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_w8.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or partial_residency or config2_full" > gpurun_out/r83_pytest.log 2>&1; tail -2 gpurun_out/r83_pytest.log
bash tools/gpurun_calls/_run33.sh
for v in base w8 w8b; do
  RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_$v.so timeout 600 python tools/bench_config5.py --frames 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5', d['frames_per_s'])"
done
