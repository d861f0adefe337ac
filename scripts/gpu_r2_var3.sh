mkdir -p gpurun_out
for v in base xc1 xc2; do
  if [ $v = base ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/var3_$v.json 2> gpurun_out/var3_$v.err
done
FSK_LIB=build/variants/xc1.so timeout 900 python -m pytest tests/test_gpu_exact.py -q -x > gpurun_out/var3_tests.log 2>&1; echo "rc $?" >> gpurun_out/var3_tests.log
timeout 600 python scripts/diag_outliers.py 64 64 64 135 training > gpurun_out/diag135.log 2>&1
