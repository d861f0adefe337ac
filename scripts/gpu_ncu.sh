# ncu captures of the step's kernels (after the same command ran clean), plus the launch list.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph"
$B > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_search_fast|k_search_escalated|k_dedup|k_emit|k_precompute|k_sort_scan" -s 8 -c 6 -o gpurun_out/r01_final_search $B > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_mlp_fwd" -s 4 -c 4 -o gpurun_out/r01_final_mlp $B > gpurun_out/ncu_mlp.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r01_final_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
