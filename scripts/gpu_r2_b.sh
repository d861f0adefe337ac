mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/r2_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-mlp > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err
timeout 600 python bench.py --backward --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/r2_c3.json 2> gpurun_out/r2_c3.err
timeout 600 python bench.py --backward --deterministic --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/r2_c3det.json 2> gpurun_out/r2_c3det.err
