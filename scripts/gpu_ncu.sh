# one ncu --set full capture of the search kernels (after the same command ran clean)
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_search_fast|k_search_escalated|k_dedup|k_emit|k_precompute" -s 7 -c 5 -o gpurun_out/prof8 $B > gpurun_out/ncu8.log 2>&1
