# production rules of round 2 (cap 8, conditioning threshold max|J~| > 5): GPU suite, C2/C3det lines,
# and the 450-scene band study + the max_iters 10 set against the default (FMA) oracle
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/jm_tests.log 2>&1; echo "rc $?" >> gpurun_out/jm_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 > gpurun_out/jm_c2.json 2> gpurun_out/jm_c2.err
for v in default detb; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --backward --deterministic --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/jm_c3det_$v.json 2> gpurun_out/jm_c3det_$v.err
done
for s in 22 52 82 112; do
  timeout 1500 python scripts/band_study.py $s $((s+30)) > gpurun_out/jm_band_$s.log 2>&1
done
BAND_MAX_ITERS=10 timeout 1500 python scripts/band_study.py 22 32 > gpurun_out/jm_band_mi10.log 2>&1
