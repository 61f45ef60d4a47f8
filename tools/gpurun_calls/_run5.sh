bash tools/gpu_iter.sh it5
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
