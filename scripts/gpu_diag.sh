timeout 600 python -m pytest tests/test_gpu_mlp.py -q -rf -s > gpurun_out/pytest_mlp.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_bwd.log 2>&1
