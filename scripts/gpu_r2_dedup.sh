mkdir -p gpurun_out
for v in default dedupold; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/dd_hash.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/dd_tests.log 2>&1; echo "rc $?" >> gpurun_out/dd_tests.log
for v in default dedupold default dedupold; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/dd_c2_$v.json 2>> gpurun_out/dd_c2_$v.err
done
