timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_all.log 2>&1
BENCH_ARGS="--no-mlp" bash scripts/gpu_variants.sh
