mkdir -p gpurun_out
BAND_POINTS=rays,training timeout 1500 python scripts/band_study.py 232 262 > gpurun_out/fc_232.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 > gpurun_out/fc_c2.json 2> gpurun_out/fc_c2.err
timeout 1500 python -m pytest tests -m gpu -q -x -k "full_bench or all_solves or exact or edges or random" > gpurun_out/fc_tests.log 2>&1; echo "rc $?" >> gpurun_out/fc_tests.log
timeout 1500 python scripts/band_study.py 202 232 > gpurun_out/fc_202.log 2>&1
