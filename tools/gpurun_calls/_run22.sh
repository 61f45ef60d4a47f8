python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r22_build.log 2>&1
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_nestlp.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config2_full or partial or randomized or deep" > gpurun_out/r22_nest_tests.log 2>&1; tail -2 gpurun_out/r22_nest_tests.log
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
