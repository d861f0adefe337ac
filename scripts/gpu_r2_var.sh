mkdir -p gpurun_out
for v in base r1m4 r1m5 r2m4 r0m5 r3m3b64; do
  if [ $v = base ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
done
timeout 900 python -m pytest tests/test_cpp_api.py tests/test_gpu_frames.py -q -x -s > gpurun_out/var_tests.log 2>&1; echo "rc $?" >> gpurun_out/var_tests.log
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe2.log 2>&1
