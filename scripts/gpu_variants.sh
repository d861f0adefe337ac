set -x
python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest12.log 2>&1
python bench.py --steps 50 --warmup 5 --cpu-seconds 3 > gpurun_out/bench12.log 2>&1
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --grid 128,128,32 --points 8000000 > gpurun_out/bench12_c5.log 2>&1
