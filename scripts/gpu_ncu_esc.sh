# ncu --set full of both float64 escalation kernels (plain f64 and exact replay)
mkdir -p gpurun_out
for v in 1 0; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:escalated<.bool.$v>" -c 1 -o gpurun_out/esc_b$v -f python scripts/precision_modes.py --steps 1 > gpurun_out/ncu_esc_b$v.log 2>&1; echo "rc $?" >> gpurun_out/ncu_esc_b$v.log
done
