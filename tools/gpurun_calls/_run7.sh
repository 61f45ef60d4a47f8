bash tools/gpu_iter.sh it7 "randomized or golden or config2 or partial"
cat gpurun_out/it7_bench.log | tail -1 | head -c 2500
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
