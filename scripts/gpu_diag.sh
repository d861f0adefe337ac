timeout 900 python -m pytest tests -m gpu -q -rf -s -k "sweep" > gpurun_out/pytest_sweep2.log 2>&1
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_step.log 2>&1
timeout 1500 python scripts/band_study.py 10 22 > gpurun_out/band2.log 2>&1
