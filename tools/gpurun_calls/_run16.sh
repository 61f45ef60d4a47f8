python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r16_build.log 2>&1
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
