# ncu captures of the step's kernels (after the same command ran clean), plus the launch list.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph"
$B > gpurun_out/ncu_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_search_fast|k_search_escalated|k_dedup|k_emit|k_precompute" -s 7 -c 5 -o gpurun_out/prof_r02 $B > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_launch.log 2>&1
