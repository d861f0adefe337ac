timeout 900 python -m pytest tests/test_gpu_edges.py -q -rf > gpurun_out/pytest_edges.log 2>&1
