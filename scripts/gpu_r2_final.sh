# Round-2 measurement set: full GPU suite, C2 default line (cpu baseline, e2e, MLP stages), C3 both
# backward modes, C4, C5 per-GPU shard, the reference arm, then ncu captures (after the plain runs).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/f2_tests.log 2>&1; echo "rc $?" >> gpurun_out/f2_tests.log
timeout 900 python bench.py > gpurun_out/f2_c2.json 2> gpurun_out/f2_c2.err
timeout 600 python bench.py --backward --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/f2_c3.json 2> gpurun_out/f2_c3.err
timeout 600 python bench.py --backward --deterministic --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/f2_c3det.json 2> gpurun_out/f2_c3det.err
timeout 900 python bench.py --poses 16 --points 1000000 --grid 64,64,64 --steps 5 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/f2_c4.json 2> gpurun_out/f2_c4.err
timeout 900 python bench.py --points 8000000 --grid 128,128,32 --steps 10 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/f2_c5.json 2> gpurun_out/f2_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f2_ref.json 2> gpurun_out/f2_ref.err
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --no-mlp --backward"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_search_fast|k_esc_start|k_search_escalated|k_dedup|k_bwd_scatter_agg|k_precompute_v" -c 6 -o gpurun_out/r02_final_search -f $B > gpurun_out/f2_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-e2e > gpurun_out/f2_ncu_l.log 2>&1
