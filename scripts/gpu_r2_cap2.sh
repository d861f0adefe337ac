# float32 cap 9: band study on the remaining seed sets, max_iters 10, and the conditioning threshold
mkdir -p gpurun_out
export FSK_LIB=build/variants/study.so FSK_ESC_CAP=9
for j in 5 6; do
  FSK_ESC_JMAX=$j timeout 600 python bench.py --no-cpu-baseline --no-mlp --no-e2e --steps 200 > gpurun_out/cap9_c2_jmax$j.json 2> gpurun_out/cap9_c2_jmax$j.err
done
FSK_ESC_JMAX=5 timeout 1500 python scripts/band_study.py 112 142 > gpurun_out/cap9_band_112_jmax5.log 2>&1
timeout 1500 python scripts/band_study.py 112 142 > gpurun_out/cap9_band_112.log 2>&1
timeout 1500 python scripts/band_study.py 52 82 > gpurun_out/cap9_band_52.log 2>&1
timeout 1500 python scripts/band_study.py 82 112 > gpurun_out/cap9_band_82.log 2>&1
BAND_MAX_ITERS=10 timeout 1500 python scripts/band_study.py 22 32 > gpurun_out/cap9_band_mi10.log 2>&1
