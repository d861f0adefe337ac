mkdir -p gpurun_out
FSK_LIB=build/variants/checked.so timeout 2400 python -m pytest tests -m gpu -q -rf -x > gpurun_out/r2_checked_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2_checked_tests.log
FSK_LIB=build/variants/checked.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/r2_checked_c2.json 2>&1; echo "rc $?" >> gpurun_out/r2_checked_c2.json
FSK_LIB=build/variants/checked.so timeout 600 python bench.py --steps 3 --warmup 3 --points 8000000 --grid 128,128,32 --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/r2_checked_c5.json 2>&1; echo "rc $?" >> gpurun_out/r2_checked_c5.json
