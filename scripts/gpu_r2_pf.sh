mkdir -p gpurun_out
for v in default nopf; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/pf_hash.log 2>&1
done
for v in default nopf default nopf; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 >> gpurun_out/pf_c2_$v.json 2>> gpurun_out/pf_c2_$v.err
  env $L timeout 600 python bench.py --points 1000000 --grid 64,64,64 --steps 20 --no-cpu-baseline --no-mlp --no-e2e >> gpurun_out/pf_c4_$v.json 2>> gpurun_out/pf_c4_$v.err
done
