# final measurement set (after the face rule) + more band-study scenes
bash scripts/gpu_r2_final.sh
BAND_POINTS=rays,uniform,training timeout 1500 python scripts/band_study.py 262 292 > gpurun_out/fb_262.log 2>&1
BAND_POINTS=rays timeout 1500 python scripts/band_study.py 292 322 > gpurun_out/fb_292.log 2>&1
