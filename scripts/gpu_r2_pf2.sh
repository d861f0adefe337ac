mkdir -p gpurun_out
for v in default pf0; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/pe_hash.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_parity.py -q -x > gpurun_out/pe_tests.log 2>&1; echo "rc $?" >> gpurun_out/pe_tests.log
for v in default pf0 pf1 pf8 pf16 default pf0; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/pe_c2_$v.json 2>> gpurun_out/pe_c2_$v.err
done
for v in default pf0; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --points 1000000 --grid 64,64,64 --steps 20 --no-cpu-baseline --no-mlp --no-e2e >> gpurun_out/pe_c4_$v.json 2>> gpurun_out/pe_c4_$v.err
done
