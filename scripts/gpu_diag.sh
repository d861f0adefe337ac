timeout 900 python -m pytest tests/test_gpu_mlp_variant.py -q -rf -s > gpurun_out/pytest_mv.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_mv.log 2>&1
