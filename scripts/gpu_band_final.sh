# 150 further scenes (seeds 52-81) with the production build and default rules (mixed = exact-replay escalation)
mkdir -p gpurun_out
timeout 3000 python scripts/band_study.py 52 82 > gpurun_out/band_final_52_82.log 2>&1
echo "rc $?" >> gpurun_out/band_final_52_82.log
