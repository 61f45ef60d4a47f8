python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r19_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_request" > gpurun_out/r19_wide.log 2>&1; tail -3 gpurun_out/r19_wide.log
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_tma.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config2_full or partial or randomized" > gpurun_out/r19_tma_tests.log 2>&1; tail -3 gpurun_out/r19_tma_tests.log
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
bash tools/ncu_metrics.sh $PWD/paper_2309_04393_b200/_variants/libresoct_base.so r19_m_base
bash tools/ncu_metrics.sh $PWD/paper_2309_04393_b200/_variants/libresoct_tma.so r19_m_tma
cat gpurun_out/r19_m_base.txt; echo ---; cat gpurun_out/r19_m_tma.txt
