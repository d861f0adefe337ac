timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -s -k "large_batch" > gpurun_out/pytest_large.log 2>&1
timeout 2400 python scripts/band_study.py 22 52 > gpurun_out/band3.log 2>&1
