python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r14_build.log 2>&1
python tools/first_frame.py > gpurun_out/r14_ff_default.log 2>&1; tail -c 1500 gpurun_out/r14_ff_default.log; echo
CUDA_MODULE_LOADING=EAGER python tools/first_frame.py > gpurun_out/r14_ff_eager.log 2>&1; tail -c 1500 gpurun_out/r14_ff_eager.log
