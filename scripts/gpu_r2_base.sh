# Round-2 baseline on a fresh box: full GPU suite, default bench line, launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r2_base_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2_base_tests.log
timeout 600 python bench.py > gpurun_out/r2_base_c2.json 2> gpurun_out/r2_base_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_base_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/r2_base_ncu.log 2>&1
echo done
