mkdir -p gpurun_out
for v in base map1 map1bpg12 map1bpg6; do
  if [ $v = base ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/map_$v.json 2> gpurun_out/map_$v.err
done
FSK_LIB=build/variants/map1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config1 or default_iters or order_independent or device_correspondence" > gpurun_out/map_tests.log 2>&1; echo "rc $?" >> gpurun_out/map_tests.log
