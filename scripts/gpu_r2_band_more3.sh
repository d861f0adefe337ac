mkdir -p gpurun_out
BAND_POINTS=rays,uniform,training timeout 1500 python scripts/band_study.py 322 352 > gpurun_out/fc3_322.log 2>&1
BAND_POINTS=rays,uniform,training timeout 1500 python scripts/band_study.py 352 382 > gpurun_out/fc3_352.log 2>&1
BAND_POINTS=rays,training timeout 1500 python scripts/band_study.py 382 412 > gpurun_out/fc3_382.log 2>&1
BAND_POINTS=uniform,training timeout 1500 python scripts/band_study.py 412 442 > gpurun_out/fc3_412.log 2>&1
