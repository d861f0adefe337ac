mkdir -p gpurun_out
for v in default sortold; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/s2_hash.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan.py -q -x > gpurun_out/s2_tests.log 2>&1; echo "rc $?" >> gpurun_out/s2_tests.log
for v in default sortold default sortold; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/s2_c2_$v.json 2>> gpurun_out/s2_c2_$v.err
done
