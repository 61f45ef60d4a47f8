bash tools/gpu_iter.sh it11 "randomized or golden or config2 or partial or render_units"
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
