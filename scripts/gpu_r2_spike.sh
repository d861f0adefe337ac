mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 > gpurun_out/sp_c2.json 2> gpurun_out/sp_c2.err
BAND_POINTS=rays,training timeout 1500 python scripts/band_study.py 382 412 > gpurun_out/sp_382.log 2>&1
BAND_POINTS=rays,uniform,training timeout 1500 python scripts/band_study.py 262 292 > gpurun_out/sp_262.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "full_bench or all_solves or exact or edges or random or parity" > gpurun_out/sp_tests.log 2>&1; echo "rc $?" >> gpurun_out/sp_tests.log
