# float32 iteration cap study: escalation rate / step time and the 150-scene band study at caps 9, 10
mkdir -p gpurun_out
for c in 8 9 10 12; do
  FSK_LIB=build/variants/study.so FSK_ESC_CAP=$c timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/cap_c2_$c.json 2> gpurun_out/cap_c2_$c.err
done
for c in 10 9; do
  FSK_LIB=build/variants/study.so FSK_ESC_CAP=$c timeout 1500 python scripts/band_study.py 22 52 > gpurun_out/cap_band_$c.log 2>&1
done
