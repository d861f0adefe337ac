# 150-scene band study with the exact-replay escalation (precision "mixed-exact")
mkdir -p gpurun_out
BAND_PRECISION=mixed-exact timeout 3000 python scripts/band_study.py 22 52 > gpurun_out/band_mixed_exact_150.log 2>&1
echo "rc $?" >> gpurun_out/band_mixed_exact_150.log
