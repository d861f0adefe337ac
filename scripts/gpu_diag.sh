timeout 600 python -m pytest tests/test_gpu_wire.py tests/test_gpu_mlp_variant.py -q -rf -s > gpurun_out/pytest_wire.log 2>&1
