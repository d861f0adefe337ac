mkdir -p gpurun_out
timeout 900 python bench.py --points 8000000 --grid 128,128,32 --steps 10 --warmup 3 --no-cpu-baseline --no-mlp > gpurun_out/f4_c5.json 2> gpurun_out/f4_c5.err
timeout 1500 python -m pytest tests/test_gpu_reference.py -q -s -k "full_bench and C5" > gpurun_out/f4_ref.log 2>&1; echo "rc $?" >> gpurun_out/f4_ref.log
timeout 900 python bench.py --impl reference --points 8000000 --grid 128,128,32 --steps 2 --warmup 1 > gpurun_out/f4_c5_ref.json 2> gpurun_out/f4_c5_ref.err
