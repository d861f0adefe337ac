mkdir -p gpurun_out
for v in base em3 em3row row sm3; do
  if [ $v = base ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/var2_$v.json 2> gpurun_out/var2_$v.err
done
FSK_LIB=build/variants/em3.so timeout 900 python -m pytest tests/test_gpu_exact.py -q -x > gpurun_out/var2_tests.log 2>&1; echo "rc $?" >> gpurun_out/var2_tests.log
