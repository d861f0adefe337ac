mkdir -p gpurun_out
for v in default nopf64; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/p6_hash.log 2>&1
done
for v in default nopf64 default nopf64; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/p6_c2_$v.json 2>> gpurun_out/p6_c2_$v.err
done
