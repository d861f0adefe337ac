mkdir -p gpurun_out
for v in default spk3 nospk default spk3 nospk; do
  if [ $v = default ]; then L=""; else L="FSK_LIB=build/variants/$v.so"; fi
  env $L timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 300 >> gpurun_out/s2p_c2_$v.json 2>> gpurun_out/s2p_c2_$v.err
done
FSK_LIB=build/variants/spk3.so BAND_POINTS=rays,training timeout 1500 python scripts/band_study.py 382 412 > gpurun_out/s2p_382.log 2>&1
FSK_LIB=build/variants/spk3.so BAND_POINTS=rays,uniform,training timeout 1500 python scripts/band_study.py 262 292 > gpurun_out/s2p_262.log 2>&1
