# ncu captures of the default step (exact-replay escalation), after the same command ran clean.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-mlp"
$B > gpurun_out/ncu_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_search_fast|k_esc_start|k_search_escalated|k_dedup" -s 8 -c 4 -o gpurun_out/r01_default_search -f $B > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01_default_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
