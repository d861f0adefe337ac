# Escalation-rule relaxation study (study build: -DFSK_ESC_REASONS -DFSK_ESC_STUDY): per-rule counts
# under each setting, then the GPU band study against the f64 oracle on a seed range.
mkdir -p gpurun_out
export FSK_LIB=build/variants/study.so
for cfg in "base" "FSK_ESC_CONV_BAND_LAST=1" "FSK_ESC_MIN_DIV=5" "FSK_ESC_CONV_BAND_LAST=1 FSK_ESC_MIN_DIV=5"; do
  echo "=== $cfg" >> gpurun_out/study_reasons.log
  env $([ "$cfg" = base ] || echo $cfg) timeout 600 python scripts/esc_reasons.py >> gpurun_out/study_reasons.log 2>&1
done
for cfg in ${BAND_CFGS:-"FSK_ESC_CONV_BAND_LAST=1 FSK_ESC_MIN_DIV=5"}; do :; done
env ${BAND_ENV:-FSK_ESC_CONV_BAND_LAST=1 FSK_ESC_MIN_DIV=5} timeout ${BAND_T:-1500} python scripts/band_study.py ${BAND_SEEDS:-22 29} > gpurun_out/study_band.log 2>&1
echo "rc $?" >> gpurun_out/study_band.log
