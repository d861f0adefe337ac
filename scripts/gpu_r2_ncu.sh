# tests subset + benches + ncu captures of the search kernels (round 2)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/r2_tests.log 2>&1; echo "rc $?" >> gpurun_out/r2_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-mlp > gpurun_out/r2_c2.json 2> gpurun_out/r2_c2.err
timeout 600 python bench.py --backward --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/r2_c3.json 2> gpurun_out/r2_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_search_fast|k_esc_start|k_search_escalated|k_dedup|k_bwd_scatter_agg|k_precompute" -c 6 -o gpurun_out/r2_search -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-mlp --backward > gpurun_out/r2_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/r2_ncu_l.log 2>&1
