mkdir -p gpurun_out
for v in default k1narrow; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/kw_hash.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/kw_tests.log 2>&1; echo "rc $?" >> gpurun_out/kw_tests.log
for v in default k1narrow default k1narrow; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --points 8000000 --grid 128,128,32 --steps 10 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e >> gpurun_out/kw_c5_$v.json 2>> gpurun_out/kw_c5_$v.err
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 >> gpurun_out/kw_c2_$v.json 2>> gpurun_out/kw_c2_$v.err
done
