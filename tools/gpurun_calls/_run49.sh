timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render_units.py tests/test_gpu_acceptance.py -m gpu -x -q > gpurun_out/r49_pytest.log 2>&1; tail -2 gpurun_out/r49_pytest.log
bash tools/gpurun_calls/_run33.sh
