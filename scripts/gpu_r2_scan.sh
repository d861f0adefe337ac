mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/sc_tests.log 2>&1; echo "rc $?" >> gpurun_out/sc_tests.log
for v in default scan3 k3shfl default scan3 k3shfl; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --backward --no-cpu-baseline --no-mlp --no-e2e --steps 200 >> gpurun_out/sc_c3_$v.json 2>> gpurun_out/sc_c3_$v.err
done
