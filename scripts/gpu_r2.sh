mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -s -k "sweep or parity or precision" > gpurun_out/pytest_sweep.log 2>&1
VARIANTS="build/variants/nocache.so" bash scripts/gpu_variants.sh
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_rule.log 2>&1
