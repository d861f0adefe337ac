timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full.log 2>&1
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
