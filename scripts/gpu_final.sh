# Round-1 measurement set: C2 default line, C3 (both backward modes), C4, C5 per-GPU shard.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
timeout 600 python bench.py --backward --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
timeout 600 python bench.py --backward --deterministic --no-cpu-baseline --no-e2e --no-mlp > gpurun_out/final_c3det.json 2> gpurun_out/final_c3det.err
timeout 900 python bench.py --poses 16 --points 1000000 --grid 64,64,64 --steps 5 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
timeout 900 python bench.py --points 8000000 --grid 128,128,32 --steps 10 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
# the same configs with the fused float64 escalation (ablation lines, FSK_SEARCH_FAST_ESC)
timeout 600 python bench.py --precision mixed-fast --no-mlp --no-cpu-baseline > gpurun_out/fused_c2.json 2> gpurun_out/fused_c2.err
timeout 900 python bench.py --precision mixed-fast --poses 16 --points 1000000 --grid 64,64,64 --steps 5 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/fused_c4.json 2> gpurun_out/fused_c4.err
