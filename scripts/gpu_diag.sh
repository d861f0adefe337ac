BENCH_ARGS="--no-mlp" bash scripts/gpu_variants.sh
