FULL=1 bash tools/gpu_iter.sh it6
rm -f gpurun_out/variants.txt
bash tools/variant_bench.sh
cat gpurun_out/variants.txt
