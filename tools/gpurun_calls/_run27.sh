python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r27_build.log 2>&1
RESOCT_LIB=$PWD/paper_2309_04393_b200/_variants/libresoct_unroll4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render_units.py -q -x > gpurun_out/r27_tests.log 2>&1; tail -2 gpurun_out/r27_tests.log
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
