# more band-study scenes with the final rules: ray samples, and a further uniform/training set
mkdir -p gpurun_out
BAND_POINTS=rays timeout 1500 python scripts/band_study.py 142 172 > gpurun_out/bm_rays_142.log 2>&1
timeout 1500 python scripts/band_study.py 172 202 > gpurun_out/bm_172.log 2>&1
BAND_MAX_ITERS=10 timeout 1500 python scripts/band_study.py 22 32 > gpurun_out/bm_mi10.log 2>&1
