mkdir -p gpurun_out
for v in default gwtile; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/bwd_hash.py >> gpurun_out/gw_hash.log 2>&1
  env $L timeout 600 python bench.py --backward --no-cpu-baseline --no-e2e --no-mlp --steps 200 >> gpurun_out/gw_c3_$v.json 2>> gpurun_out/gw_c3_$v.err
done
