mkdir -p gpurun_out
for v in default noffma2; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/ffma2_hash.log 2>&1
done
for v in default noffma2 default noffma2; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 >> gpurun_out/ffma2_c2_$v.json 2>> gpurun_out/ffma2_c2_$v.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/ffma2_tests.log 2>&1; echo "rc $?" >> gpurun_out/ffma2_tests.log
