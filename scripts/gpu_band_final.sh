# 150 further scenes with the production build and default rules (mixed = exact-replay escalation)
mkdir -p gpurun_out
A=${BAND_FROM:-82}; B=${BAND_TO:-112}
timeout 3000 python scripts/band_study.py $A $B > gpurun_out/band_final_${A}_${B}.log 2>&1
echo "rc $?" >> gpurun_out/band_final_${A}_${B}.log
