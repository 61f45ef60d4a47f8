for v in nestonly sub32only; do
  echo "== $v"; RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
done
