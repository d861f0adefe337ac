mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/st_tests.log 2>&1; echo "rc $?" >> gpurun_out/st_tests.log
for v in 1 0 1 0; do
  FSK_PIPE_STAGE=$v timeout 600 python bench.py --no-cpu-baseline --no-mlp --steps 100 >> gpurun_out/st_c2_$v.json 2>> gpurun_out/st_c2_$v.err
done
for v in 1 0; do
  FSK_PIPE_STAGE=$v timeout 900 python bench.py --poses 16 --points 1000000 --grid 64,64,64 --steps 5 --warmup 3 --no-cpu-baseline --no-mlp >> gpurun_out/st_c4_$v.json 2>> gpurun_out/st_c4_$v.err
done
