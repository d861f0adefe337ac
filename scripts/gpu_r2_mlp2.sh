mkdir -p gpurun_out
for v in default mlpnostream default mlpnostream; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 >> gpurun_out/ml2_$v.json 2>> gpurun_out/ml2_$v.err
done
