mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/so_tests.log 2>&1; echo "rc $?" >> gpurun_out/so_tests.log
for v in default sort4; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/variant_hash.py >> gpurun_out/so_hash.log 2>&1
done
for v in default sort4 default sort4; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/so_c2_$v.json 2>> gpurun_out/so_c2_$v.err
  env $L timeout 600 python bench.py --points 8000000 --grid 128,128,32 --steps 10 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e >> gpurun_out/so_c5_$v.json 2>> gpurun_out/so_c5_$v.err
done
FSK_PIPE_GRAPH=1 timeout 600 python bench.py --no-cpu-baseline --no-mlp --steps 100 > gpurun_out/so_c2_e2e.json 2> gpurun_out/so_c2_e2e.err
