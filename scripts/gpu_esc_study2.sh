# "converged on the cap iteration" rule study (study build): per-rule counts, then the band study on seeds 52-81
mkdir -p gpurun_out
export FSK_LIB=build/variants/study.so
for v in 1 2; do echo "=== capconv $v" >> gpurun_out/study_capconv_reasons.log; FSK_ESC_CAPCONV=$v timeout 600 python scripts/esc_reasons.py >> gpurun_out/study_capconv_reasons.log 2>&1; done
FSK_ESC_CAPCONV=2 timeout 1500 python scripts/band_study.py 52 82 > gpurun_out/study_band_capconv2.log 2>&1
FSK_ESC_CAPCONV=1 timeout 1500 python scripts/band_study.py 52 82 > gpurun_out/study_band_capconv1.log 2>&1
echo done >> gpurun_out/study_band_capconv1.log
