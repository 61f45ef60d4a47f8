for v in base run4; do
  RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_$v.so timeout 600 python tools/bench_config5.py --frames 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['frames_per_s'], d['ms_per_frame_p50'])"
done
