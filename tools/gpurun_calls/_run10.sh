python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r10_build.log 2>&1
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
