timeout 600 python scripts/diag_outliers.py 128 128 32 10 uniform > gpurun_out/diag1.log 2>&1
