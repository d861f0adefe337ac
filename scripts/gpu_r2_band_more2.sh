mkdir -p gpurun_out
timeout 1500 python scripts/band_study.py 202 232 > gpurun_out/bm2_202.log 2>&1
BAND_POINTS=rays,training timeout 1500 python scripts/band_study.py 232 262 > gpurun_out/bm2_232.log 2>&1
