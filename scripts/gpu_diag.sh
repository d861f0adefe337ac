timeout 600 python -m pytest tests/test_gpu_mlp.py -q -rf -s -x > gpurun_out/pytest_mlp.log 2>&1
