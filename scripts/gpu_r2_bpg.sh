mkdir -p gpurun_out
for v in default bpg4 bpg6 bpg12 map0 default; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/bp_c2_$v.json 2>> gpurun_out/bp_c2_$v.err
done
