timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_mlp_variant.py -q -rf > gpurun_out/pytest_mlp2.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mlp2.log 2>&1
