mkdir -p gpurun_out
for v in default detord; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 300 python scripts/bwd_hash.py >> gpurun_out/d2_hash.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist_det.py tests/test_gpu_multi.py -q -x > gpurun_out/d2_tests.log 2>&1; echo "rc $?" >> gpurun_out/d2_tests.log
timeout 600 python bench.py --backward --deterministic --no-cpu-baseline --no-e2e --no-mlp --steps 200 > gpurun_out/d2_c3det.json 2> gpurun_out/d2_c3det.err
