timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "precision or config1" > gpurun_out/pytest_stats.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/bench_stats.log 2>&1
