mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_frames.py tests/test_lib_exports.py -q -x > gpurun_out/df_tests.log 2>&1; echo "rc $?" >> gpurun_out/df_tests.log
for v in "" "--no-stage-frames" "" "--no-stage-frames"; do
  timeout 900 python bench.py --poses 16 --points 1000000 --grid 64,64,64 --steps 5 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e $v >> gpurun_out/df_c4.json 2>> gpurun_out/df_c4.err
done
