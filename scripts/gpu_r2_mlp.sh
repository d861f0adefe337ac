mkdir -p gpurun_out
for v in default mlp512; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_gpu_mlp_variant.py -q -x > gpurun_out/ml_tests_$v.log 2>&1; echo "rc $?" >> gpurun_out/ml_tests_$v.log
done
for v in default mlp512 default mlp512; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 50 >> gpurun_out/ml_c2_$v.json 2>> gpurun_out/ml_c2_$v.err
done
